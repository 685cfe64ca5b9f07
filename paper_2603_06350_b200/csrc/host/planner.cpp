// planner.cpp — host-side C++ for the B200 MoE layer: keyed RNG, popularity
// profile and routing stand-in, load predictor, Algorithm-1 scaler,
// Algorithm-2 placer + keep-alive registry, the analytic forward model and the
// reference baselines the bench reports beside the measured layer.
//
// Written fresh for this build against the reference's documented behaviour
// (SPEC.md, Alg. 1/2).  Where the reference takes a decision on a
// floating-point expression, the same expression and evaluation order are used
// so plans come out bit-identical; tests/test_planner_parity.py checks that
// against the compiled reference (oracle/_ref) on thousands of random cases.
#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <string>

#include "host/moeless_api.hpp"

namespace moeless {

using std::int64_t;
using std::to_string;

// =================================================================== rng
// reference rng.hpp:12-25
std::uint64_t mix64(std::uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

std::mt19937_64 keyed_engine(std::uint64_t seed, std::uint64_t a, std::uint64_t b,
                             std::uint64_t tag) {
  const std::uint64_t k = mix64(tag);
  return std::mt19937_64(mix64(seed ^ mix64(a ^ mix64(b ^ k))));
}

// ================================================================ specs
void ClusterSpec::validate() const {
  auto need = [](bool ok, const char* msg) { if (!ok) throw std::invalid_argument(msg); };
  need(gpu_count >= 1, "gpu_count must be >= 1");
  need(gpu_mem_capacity_mb > 0, "gpu_mem_capacity_mb must be > 0");
  need(alpha_ms_per_token >= 0, "alpha_ms_per_token must be >= 0");
  need(beta_ms_per_token >= 0, "beta_ms_per_token must be >= 0");
  need(t_misc_ms >= 0, "t_misc_ms must be >= 0");
  need(m_misc_mb >= 0, "m_misc_mb must be >= 0");
}

void ModelSpec::validate() const {
  auto need = [](bool ok, const char* msg) { if (!ok) throw std::invalid_argument(msg); };
  need(num_layers >= 1, "num_layers must be >= 1");
  need(experts_per_layer >= 1, "experts_per_layer must be >= 1");
  need(top_k >= 1 && top_k <= experts_per_layer, "top_k must be in [1, experts_per_layer]");
  need(expert_mem_mb > 0, "expert_mem_mb must be > 0");
  need(layer_mem_cap_mb >= 0, "layer_mem_cap_mb must be >= 0");
}

// ============================================================ workload
namespace {
constexpr std::uint64_t kTagRoute = 0x726f757465ULL;  // "route"
constexpr std::uint64_t kTagPerm = 0x7065726dULL;     // "perm"
constexpr std::uint64_t kTagNoise = 0x6e6f697379ULL;  // "noisy"

// In-place Fisher-Yates driven by raw 64-bit draws (cross-platform stable).
void shuffle_in_place(std::vector<int>& v, std::mt19937_64& eng) {
  for (int i = static_cast<int>(v.size()) - 1; i >= 1; --i) {
    const auto j = static_cast<int>(eng() % static_cast<std::uint64_t>(i + 1));
    std::swap(v[i], v[j]);
  }
}

double zipf_mass(int rank, double s) { return 1.0 / std::pow(static_cast<double>(rank + 1), s); }
}  // namespace

PopularityProfile make_popularity_profile(int experts, int layers, double zipf_exponent,
                                          std::uint64_t seed, bool shared_permutation,
                                          int drift_period, double zipf_exponent_decode) {
  if (experts < 1) throw std::invalid_argument("experts must be >= 1");
  if (layers < 1) throw std::invalid_argument("layers must be >= 1");
  if (zipf_exponent < 0) throw std::invalid_argument("zipf exponent must be >= 0");
  if (drift_period < 0) throw std::invalid_argument("drift_period must be >= 0");
  PopularityProfile prof;
  prof.zipf_exponent = zipf_exponent;
  prof.zipf_exponent_decode = zipf_exponent_decode;
  prof.drift_period = drift_period;
  prof.perm_seed = seed;
  for (int l = 0; l < layers; ++l) {
    std::vector<int> perm(experts);
    std::iota(perm.begin(), perm.end(), 0);
    auto eng = keyed_engine(seed, shared_permutation ? 0u : static_cast<std::uint64_t>(l), 0, kTagPerm);
    shuffle_in_place(perm, eng);
    prof.rank_to_expert.push_back(std::move(perm));
  }
  return prof;
}

std::vector<int> effective_permutation(const PopularityProfile& profile, int layer, long iteration) {
  if (layer < 0 || layer >= profile.num_layers()) throw std::invalid_argument("layer out of range");
  std::vector<int> perm = profile.rank_to_expert[layer];
  if (profile.drift_period > 0) {
    const long epoch = iteration / profile.drift_period;
    if (epoch > 0) {
      auto eng = keyed_engine(profile.perm_seed, static_cast<std::uint64_t>(epoch),
                              static_cast<std::uint64_t>(layer), kTagPerm + 1);
      shuffle_in_place(perm, eng);
    }
  }
  return perm;
}

std::vector<double> popularity_weights(const PopularityProfile& profile, int layer, long iteration,
                                       Phase phase) {
  const std::vector<int> perm = effective_permutation(profile, layer, iteration);
  const double s = profile.exponent_for(phase);
  const int n = static_cast<int>(perm.size());
  double z = 0.0;
  for (int r = 0; r < n; ++r) z += zipf_mass(r, s);
  std::vector<double> w(n, 0.0);
  for (int r = 0; r < n; ++r) w[perm[r]] = zipf_mass(r, s) / z;
  return w;
}

LoadVector route_tokens(const IterationBatch& batch, int layer, const PopularityProfile& profile,
                        int top_k, int experts, std::uint64_t seed) {
  if (experts != profile.num_experts()) throw std::invalid_argument("expert count does not match profile");
  if (top_k < 1 || top_k > experts) throw std::invalid_argument("top_k must be in [1, experts]");
  if (batch.token_count < 0) throw std::invalid_argument("token_count must be >= 0");
  const std::vector<int> perm = effective_permutation(profile, layer, batch.iteration);
  const double s = profile.exponent_for(batch.phase);
  std::vector<double> cdf(experts);
  double z = 0.0;
  for (int r = 0; r < experts; ++r) cdf[r] = (z += zipf_mass(r, s));

  LoadVector out;
  out.layer = layer;
  out.loads.assign(experts, 0);
  auto eng = keyed_engine(seed, static_cast<std::uint64_t>(batch.iteration),
                          static_cast<std::uint64_t>(layer), kTagRoute);
  std::vector<int> taken;
  taken.reserve(top_k);
  for (int64_t t = 0; t < batch.token_count; ++t) {
    taken.clear();
    while (static_cast<int>(taken.size()) < top_k) {
      const double u = uniform01(eng) * z;
      const auto rank = static_cast<int>(std::lower_bound(cdf.begin(), cdf.end(), u) - cdf.begin());
      const int e = perm[std::min(rank, experts - 1)];
      if (std::find(taken.begin(), taken.end(), e) != taken.end()) continue;  // distinct top-k
      taken.push_back(e);
      ++out.loads[e];
    }
  }
  return out;
}

// =========================================================== predictor
double PredictorProfile::effective_accuracy(int layer) const {
  if (layer < 0 || layer >= static_cast<int>(per_layer_accuracy.size()))
    throw std::invalid_argument("layer outside accuracy profile");
  const double a = per_layer_accuracy[layer] - distance_decay * std::max(0, distance - 1);
  return std::clamp(a, 0.0, 1.0);
}

void PredictorProfile::validate(int num_layers) const {
  if (distance < 0) throw std::invalid_argument("prediction distance must be >= 0");
  if (kind != PredictorKind::historical) {
    if (static_cast<int>(per_layer_accuracy.size()) != num_layers)
      throw std::invalid_argument("accuracy profile must list one value per layer");
    for (double a : per_layer_accuracy)
      if (!(a >= 0.0 && a <= 1.0)) throw std::invalid_argument("per-layer accuracy must be in [0, 1]");
  }
  if (accuracy_threshold < 0.0 || accuracy_threshold > 1.0)
    throw std::invalid_argument("accuracy_threshold must be in [0, 1]");
  if (distance_decay < 0.0) throw std::invalid_argument("distance_decay must be >= 0");
  if (history_window < 1) throw std::invalid_argument("history_window must be >= 1");
}

PredictorProfile make_ramp_profile(int num_layers, double first, double last) {
  if (num_layers < 1) throw std::invalid_argument("num_layers must be >= 1");
  PredictorProfile p;
  p.per_layer_accuracy.resize(num_layers);
  p.fine_tuned.assign(num_layers, false);
  for (int l = 0; l < num_layers; ++l) {
    const double frac = num_layers == 1 ? 0.0 : static_cast<double>(l) / (num_layers - 1);
    p.per_layer_accuracy[l] = first + (last - first) * frac;
  }
  return p;
}

namespace {

std::vector<int64_t> spread_uniform(int64_t total, int experts) {
  std::vector<int64_t> v(experts);
  for (int e = 0; e < experts; ++e) v[e] = total / experts + (e < total % experts ? 1 : 0);
  return v;
}

// Token-level noise: each routed token keeps its expert with probability a,
// otherwise it is re-drawn from the popularity CDF (totals preserved).
LoadVector noisy_forecast(const LoadVector& actual, double a, long iteration, std::uint64_t seed,
                          const std::vector<double>& popularity) {
  const int n = static_cast<int>(actual.loads.size());
  std::vector<double> w = popularity.empty() ? std::vector<double>(n, 1.0 / n) : popularity;
  if (static_cast<int>(w.size()) != n) throw std::invalid_argument("popularity weights do not match expert count");
  std::vector<double> cdf(n);
  double z = 0.0;
  for (int e = 0; e < n; ++e) {
    if (w[e] < 0) throw std::invalid_argument("negative popularity weight");
    cdf[e] = (z += w[e]);
  }
  if (z <= 0) throw std::invalid_argument("popularity weights sum to zero");
  auto eng = keyed_engine(seed, static_cast<std::uint64_t>(iteration),
                          static_cast<std::uint64_t>(actual.layer), kTagNoise);
  LoadVector out{actual.layer, std::vector<int64_t>(n, 0)};
  for (int e = 0; e < n; ++e)
    for (int64_t i = 0; i < actual.loads[e]; ++i) {
      if (uniform01(eng) < a) { ++out.loads[e]; continue; }
      const double u = uniform01(eng) * z;
      const auto dst = static_cast<int>(std::lower_bound(cdf.begin(), cdf.end(), u) - cdf.begin());
      ++out.loads[std::min(dst, n - 1)];
    }
  return out;
}

// Mean of the newest `window` vectors, rescaled to the known total with
// largest-remainder rounding (ties to the lower expert, leftovers cyclic).
LoadVector window_forecast(int64_t total, int layer, int experts,
                           const std::vector<LoadVector>& history, int window, bool* fallback) {
  LoadVector out{layer, {}};
  const int used = std::min<int>(window, static_cast<int>(history.size()));
  std::vector<double> mean(experts, 0.0);
  for (int i = 0; i < used; ++i) {
    const LoadVector& h = history[history.size() - 1 - i];
    if (static_cast<int>(h.loads.size()) != experts)
      throw std::invalid_argument("history vector has wrong expert count");
    for (int e = 0; e < experts; ++e) mean[e] += static_cast<double>(h.loads[e]);
  }
  double mass = 0.0;
  if (used > 0)
    for (int e = 0; e < experts; ++e) { mean[e] /= used; mass += mean[e]; }
  if (used == 0 || mass <= 0.0) {
    if (fallback) *fallback = true;
    out.loads = spread_uniform(total, experts);
    return out;
  }
  out.loads.assign(experts, 0);
  std::vector<std::pair<double, int>> frac(experts);
  int64_t given = 0;
  for (int e = 0; e < experts; ++e) {
    const double exact = mean[e] / mass * static_cast<double>(total);
    out.loads[e] = static_cast<int64_t>(exact);
    given += out.loads[e];
    frac[e] = {exact - static_cast<double>(out.loads[e]), e};
  }
  std::sort(frac.begin(), frac.end(), [](const auto& x, const auto& y) {
    return x.first != y.first ? x.first > y.first : x.second < y.second;
  });
  for (int64_t i = 0; i < total - given; ++i) ++out.loads[frac[i % frac.size()].second];
  return out;
}

}  // namespace

LoadVector predict(const LoadVector& actual_future, const std::vector<LoadVector>& history,
                   const PredictorProfile& profile, long iteration, std::uint64_t seed,
                   const std::vector<double>& popularity, bool* bootstrap_fallback) {
  if (bootstrap_fallback) *bootstrap_fallback = false;
  if (actual_future.loads.empty()) throw std::invalid_argument("empty load vector");
  for (int64_t v : actual_future.loads)
    if (v < 0) throw std::invalid_argument("negative load");
  switch (profile.kind) {
    case PredictorKind::oracle:
      return actual_future;
    case PredictorKind::noisy:
      return noisy_forecast(actual_future, profile.effective_accuracy(actual_future.layer), iteration,
                            seed, popularity);
    case PredictorKind::historical:
      return window_forecast(actual_future.total(), actual_future.layer,
                             static_cast<int>(actual_future.loads.size()), history,
                             profile.history_window, bootstrap_fallback);
  }
  throw std::logic_error("unknown predictor kind");
}

double measure_accuracy(const LoadVector& predicted, const LoadVector& actual) {
  if (predicted.loads.size() != actual.loads.size())
    throw std::invalid_argument("vectors differ in expert count");
  long double tot_a = 0.0L, tot_p = 0.0L;
  for (std::size_t e = 0; e < actual.loads.size(); ++e) {
    if (predicted.loads[e] < 0 || actual.loads[e] < 0) throw std::invalid_argument("negative load");
    tot_a += actual.loads[e];
    tot_p += predicted.loads[e];
  }
  if (tot_a == 0.0L) return tot_p == 0.0L ? 1.0 : 0.0;
  if (tot_p == 0.0L) return 0.0;
  const long double k = tot_a / tot_p;
  long double hit = 0.0L;
  for (std::size_t e = 0; e < actual.loads.size(); ++e)
    hit += std::min<long double>(predicted.loads[e] * k, static_cast<long double>(actual.loads[e]));
  return static_cast<double>(hit / tot_a);
}

void apply_layer_aware_finetuning(PredictorProfile& profile) {
  if (profile.kind != PredictorKind::noisy)
    throw std::invalid_argument("fine-tuning applies to the noisy predictor only");
  if (profile.fine_tuned.size() != profile.per_layer_accuracy.size())  // a mismatched mask restarts
    profile.fine_tuned.assign(profile.per_layer_accuracy.size(), false);
  for (std::size_t l = 0; l < profile.per_layer_accuracy.size(); ++l)
    if (profile.per_layer_accuracy[l] < profile.accuracy_threshold) {
      profile.per_layer_accuracy[l] = profile.accuracy_threshold;
      profile.fine_tuned[l] = true;
    }
}

// ============================================================== scaler
namespace {
constexpr double kCvSlack = 1e-9;

// CV of the per-replica share multiset (each expert contributes its share
// counts[e] times).  Same summation order as the reference (scaler.cpp:20-39)
// so borderline stop decisions agree bit for bit.
double replica_share_cv(const std::vector<int64_t>& loads, const std::vector<int>& counts,
                        bool skip_zero) {
  double mass = 0.0;
  long slots = 0;
  for (std::size_t e = 0; e < loads.size(); ++e) {
    if (skip_zero && loads[e] == 0) continue;
    mass += static_cast<double>(loads[e]);
    slots += counts[e];
  }
  if (slots == 0) return 0.0;
  const double mu = mass / slots;
  if (mu == 0.0) return 0.0;
  double ss = 0.0;
  for (std::size_t e = 0; e < loads.size(); ++e) {
    if (skip_zero && loads[e] == 0) continue;
    const double dev = static_cast<double>(loads[e]) / counts[e] - mu;
    ss += counts[e] * dev * dev;
  }
  return std::sqrt(ss / slots) / mu;
}

// Expert whose per-replica share is largest; ties go to the lowest index.
int heaviest(const std::vector<int64_t>& loads, const std::vector<int>& counts) {
  int best = 0;
  for (int e = 1; e < static_cast<int>(loads.size()); ++e)
    if (Rational(loads[best], counts[best]) < Rational(loads[e], counts[e])) best = e;
  return best;
}
}  // namespace

ScalingPlan scale_experts(const LoadVector& predicted, const ModelSpec& model,
                          const ScalerConfig& config, ScaleTrace* trace) {
  model.validate();
  if (config.cv_threshold < 0) throw std::invalid_argument("cv_threshold must be >= 0");
  const int n = static_cast<int>(predicted.loads.size());
  if (n == 0) throw std::invalid_argument("load vector is empty");
  if (n != model.experts_per_layer) throw std::invalid_argument("load vector does not match experts_per_layer");
  for (int64_t v : predicted.loads)
    if (v < 0) throw std::invalid_argument("negative predicted load");

  ScalingPlan plan;
  plan.layer = predicted.layer;
  plan.replica_counts.assign(n, 1);
  plan.expert_mem_mb = model.expert_mem_mb;
  const auto& w = predicted.loads;
  double cv = replica_share_cv(w, plan.replica_counts, config.exclude_zero_loads_from_cv);
  // Algorithm 1: keep splitting the heaviest replica while memory allows and
  // the share distribution is still too uneven.
  while (plan.alloc_mem_mb + model.expert_mem_mb <= model.layer_mem_cap_mb && cv > config.cv_threshold) {
    const int e = heaviest(w, plan.replica_counts);
    ++plan.replica_counts[e];
    plan.alloc_mem_mb += model.expert_mem_mb;
    cv = replica_share_cv(w, plan.replica_counts, config.exclude_zero_loads_from_cv);
    if (trace) {
      const int top = heaviest(w, plan.replica_counts);
      trace->split_expert.push_back(e);
      trace->max_share.push_back(Rational(w[top], plan.replica_counts[top]));
      trace->cv.push_back(cv);
    }
  }
  for (int e = 0; e < n; ++e)
    for (int r = 0; r < plan.replica_counts[e]; ++r)
      plan.shares.push_back({e, r, Rational(w[e], plan.replica_counts[e])});
  return plan;
}

VerifyReport verify_plan(const ScalingPlan& plan, const LoadVector& predicted,
                         const ModelSpec& model, const ScalerConfig& config) {
  VerifyReport rep;
  auto bad = [&rep](std::string msg) { rep.ok = false; rep.issues.push_back(std::move(msg)); };
  const int n = static_cast<int>(predicted.loads.size());
  if (static_cast<int>(plan.replica_counts.size()) != n) {
    bad("replica_counts has " + to_string(plan.replica_counts.size()) + " entries for " + to_string(n) + " experts");
    return rep;
  }
  for (int e = 0; e < n; ++e)
    if (plan.replica_counts[e] < 1) bad("expert " + to_string(e) + " has replica count " + to_string(plan.replica_counts[e]));
  if (!rep.ok) return rep;

  std::vector<std::vector<const ReplicaShare*>> per(n);
  for (const auto& s : plan.shares) {
    if (s.expert < 0 || s.expert >= n) {
      bad("share entry names unknown expert " + to_string(s.expert));
      return rep;
    }
    per[s.expert].push_back(&s);
  }
  for (int e = 0; e < n; ++e) {
    const int cnt = plan.replica_counts[e];
    if (static_cast<int>(per[e].size()) != cnt) {
      bad("expert " + to_string(e) + " lists " + to_string(per[e].size()) + " shares for " + to_string(cnt) + " replicas");
      continue;
    }
    std::vector<char> seen(cnt, 0);
    Rational sum(0);
    bool uniform = true;
    for (const ReplicaShare* s : per[e]) {
      if (s->ordinal < 0 || s->ordinal >= cnt || seen[s->ordinal]) {
        bad("expert " + to_string(e) + " has duplicate or out-of-range ordinal " + to_string(s->ordinal));
        uniform = false;
        break;
      }
      seen[s->ordinal] = 1;
      sum = sum + s->share;
      uniform = uniform && s->share == per[e][0]->share;
    }
    if (!uniform) { bad("expert " + to_string(e) + " has unequal replica shares"); continue; }
    if (sum != Rational(predicted.loads[e], 1))
      bad("expert " + to_string(e) + " shares sum to " + to_string(sum.to_double()) + ", load is " + to_string(predicted.loads[e]));
  }
  const double expect = (plan.total_replicas() - n) * model.expert_mem_mb;
  if (std::abs(plan.alloc_mem_mb - expect) > 1e-6)
    bad("alloc_mem_mb " + to_string(plan.alloc_mem_mb) + " does not match replicas (" + to_string(expect) + ")");
  if (plan.alloc_mem_mb > model.layer_mem_cap_mb + 1e-6) bad("alloc_mem_mb exceeds layer_mem_cap_mb");
  const double cv = replica_share_cv(predicted.loads, plan.replica_counts, config.exclude_zero_loads_from_cv);
  const bool exhausted = plan.alloc_mem_mb + model.expert_mem_mb > model.layer_mem_cap_mb;
  if (cv > config.cv_threshold + kCvSlack && !exhausted)
    bad("plan stopped with CV " + to_string(cv) + " above threshold and budget left");
  return rep;
}

// ============================================================== placer
ReplicaRegistry::ReplicaRegistry(int keep_alive_iters) : keep_alive_(keep_alive_iters) {
  if (keep_alive_iters < 0) throw std::invalid_argument("keep_alive_iters must be >= 0");
}

std::optional<int> ReplicaRegistry::lookup(int layer, int expert, int ordinal, long iteration) const {
  auto it = live_.find({layer, expert, ordinal});
  if (it == live_.end() || iteration - it->second.last_used > keep_alive_) return std::nullopt;
  return it->second.gpu;
}

void ReplicaRegistry::record(int layer, int expert, int ordinal, int gpu, long iteration) {
  live_[{layer, expert, ordinal}] = Entry{gpu, iteration};
}

void ReplicaRegistry::retire(int layer, const Placement& placement, long iteration) {
  std::erase_if(live_, [&](const auto& kv) {
    const auto& [l, e, r] = kv.first;
    if (l != layer) return false;
    const bool gone = e >= static_cast<int>(placement.gpu_for.size()) ||
                      r >= static_cast<int>(placement.gpu_for[e].size());
    return gone || iteration - kv.second.last_used > keep_alive_;
  });
}

PlaceResult place_experts(const ScalingPlan& plan, const ClusterSpec& cluster,
                          const ReplicaRegistry& registry, long iteration,
                          const PlacerOptions& options) {
  cluster.validate();
  const int G = cluster.gpu_count;
  const int n = static_cast<int>(plan.replica_counts.size());
  if (n == 0) throw std::invalid_argument("plan covers no experts");
  const double cap = cluster.gpu_mem_capacity_mb;
  if (plan.total_replicas() * plan.expert_mem_mb > G * cap + 1e-9)
    throw std::runtime_error("plan memory exceeds aggregate cluster capacity for layer " + to_string(plan.layer));

  PlaceResult res;
  Placement& pl = res.placement;
  pl.layer = plan.layer;
  pl.per_gpu_mem_mb.assign(G, 0.0);
  for (int e = 0; e < n; ++e) pl.gpu_for.emplace_back(plan.replica_counts[e], -1);

  // Algorithm 2: heaviest share first (ties: expert, then ordinal).
  std::vector<ReplicaShare> order(plan.shares);
  std::sort(order.begin(), order.end(), [](const ReplicaShare& x, const ReplicaShare& y) {
    if (x.share != y.share) return y.share < x.share;
    return x.expert != y.expert ? x.expert < y.expert : x.ordinal < y.ordinal;
  });
  const double m = plan.expert_mem_mb;
  auto fits = [&](int g) { return pl.per_gpu_mem_mb[g] + m <= cap + 1e-9; };
  std::vector<double> queue(G, 0.0);
  for (const ReplicaShare& rs : order) {
    const double sh = rs.share.to_double();
    const double add = options.beta_ms_per_token * sh + (options.load_includes_compute ? options.alpha_ms_per_token * sh : 0.0);
    int g = -1;
    bool warm = false;
    if (auto prior = registry.lookup(plan.layer, rs.expert, rs.ordinal, iteration);
        prior && *prior >= 0 && *prior < G && fits(*prior)) {
      g = *prior;
      warm = true;
    } else {
      for (int c = 0; c < G; ++c)  // join the shortest queue with room
        if (fits(c) && (g < 0 || queue[c] < queue[g])) g = c;
      if (g < 0)
        throw std::runtime_error("no GPU has memory for replica (" + to_string(rs.expert) + "," +
                                 to_string(rs.ordinal) + ") of layer " + to_string(plan.layer));
    }
    pl.gpu_for[rs.expert][rs.ordinal] = g;
    pl.per_gpu_mem_mb[g] += m;
    queue[g] += add;
    (warm ? res.warm_count : res.cold_count)++;
  }
  for (int e = 0; e < n; ++e)
    for (int r = 0; r < plan.replica_counts[e]; ++r)
      if (pl.gpu_for[e][r] < 0)
        throw std::runtime_error("plan share list misses replica (" + to_string(e) + "," + to_string(r) + ")");
  return res;
}

void update_registry(ReplicaRegistry& registry, const Placement& placement, long iteration) {
  for (int e = 0; e < static_cast<int>(placement.gpu_for.size()); ++e)
    for (int r = 0; r < static_cast<int>(placement.gpu_for[e].size()); ++r)
      registry.record(placement.layer, e, r, placement.gpu_for[e][r], iteration);
  registry.retire(placement.layer, placement, iteration);
}

// ========================================================== cost model
double replica_time(double load_share_tokens, double alpha_ms_per_token) {
  if (load_share_tokens < 0) throw std::invalid_argument("load share must be >= 0");
  if (alpha_ms_per_token < 0) throw std::invalid_argument("alpha must be >= 0");
  return alpha_ms_per_token * load_share_tokens;
}

namespace {
// Per-GPU sum of share_of(e, r) over hosted replicas, after checking that every
// replica of the plan sits on exactly one valid GPU.
template <class F>
std::vector<double> hosted_load(const ScalingPlan& plan, const Placement& pl, F&& share_of) {
  const int G = pl.gpu_count();
  if (G < 1) throw std::invalid_argument("placement covers no GPUs");
  if (pl.gpu_for.size() != plan.replica_counts.size())
    throw std::invalid_argument("placement does not match plan: expert count differs");
  std::vector<double> acc(G, 0.0);
  for (std::size_t e = 0; e < plan.replica_counts.size(); ++e) {
    if (static_cast<int>(pl.gpu_for[e].size()) != plan.replica_counts[e])
      throw std::invalid_argument("unplaced or doubly-placed replica for expert " + to_string(e));
    for (int r = 0; r < plan.replica_counts[e]; ++r) {
      const int g = pl.gpu_for[e][r];
      if (g < 0 || g >= G)
        throw std::invalid_argument("replica (" + to_string(e) + "," + to_string(r) + ") placed on invalid GPU " + to_string(g));
      acc[g] += share_of(static_cast<int>(e), r);
    }
  }
  return acc;
}
}  // namespace

std::vector<double> gpu_comm_times(const ScalingPlan& plan, const Placement& placement,
                                   double beta_ms_per_token) {
  if (beta_ms_per_token < 0) throw std::invalid_argument("beta must be >= 0");
  std::vector<std::vector<double>> sh(plan.replica_counts.size());
  for (std::size_t e = 0; e < sh.size(); ++e) sh[e].assign(std::max(plan.replica_counts[e], 0), -1.0);
  for (const auto& s : plan.shares) {
    if (s.expert < 0 || s.expert >= static_cast<int>(sh.size()) || s.ordinal < 0 ||
        s.ordinal >= static_cast<int>(sh[s.expert].size()))
      throw std::invalid_argument("plan share list names replica (" + to_string(s.expert) + "," +
                                  to_string(s.ordinal) + ") outside replica_counts");
    sh[s.expert][s.ordinal] = s.share.to_double();
  }
  for (std::size_t e = 0; e < sh.size(); ++e)
    for (std::size_t r = 0; r < sh[e].size(); ++r)
      if (sh[e][r] < 0)
        throw std::invalid_argument("plan has no share for replica (" + to_string(e) + "," + to_string(r) + ")");
  auto v = hosted_load(plan, placement, [&](int e, int r) { return sh[e][r]; });
  for (double& x : v) x *= beta_ms_per_token;
  return v;
}

LayerMetrics layer_forward_time(const ScalingPlan& plan, const Placement& placement,
                                const LoadVector& actual, const ClusterSpec& cluster,
                                const ModelSpec& model) {
  cluster.validate();
  if (actual.loads.size() != plan.replica_counts.size())
    throw std::invalid_argument("actual load vector does not match plan expert count");
  std::vector<double> per_replica(plan.replica_counts.size());
  double slowest = 0.0;
  for (std::size_t e = 0; e < per_replica.size(); ++e) {
    if (plan.replica_counts[e] < 1) throw std::invalid_argument("expert " + to_string(e) + " has no replica");
    if (actual.loads[e] < 0) throw std::invalid_argument("negative actual load");
    per_replica[e] = static_cast<double>(actual.loads[e]) / plan.replica_counts[e];
    slowest = std::max(slowest, per_replica[e]);
  }
  const auto hosted = hosted_load(plan, placement, [&](int e, int) { return per_replica[e]; });
  const double busiest = hosted.empty() ? 0.0 : *std::max_element(hosted.begin(), hosted.end());
  LayerMetrics m;
  m.compute_ms = cluster.alpha_ms_per_token * slowest;
  m.comm_ms = cluster.beta_ms_per_token * std::max(0.0, busiest);
  m.forward_ms = m.compute_ms + 2.0 * m.comm_ms + cluster.t_misc_ms;
  m.replica_count = plan.total_replicas();
  m.mem_mb = m.replica_count * model.expert_mem_mb;
  m.cost_mb_ms = (m.compute_ms + 2.0 * m.comm_ms) * m.mem_mb + cluster.t_misc_ms * cluster.m_misc_mb;
  return m;
}

double coefficient_of_variation(const std::vector<double>& values) {
  if (values.empty()) throw std::invalid_argument("CV of an empty sample");
  double sum = 0.0;
  for (double v : values) sum += v;
  const double mu = sum / values.size();
  if (mu == 0.0) return 0.0;
  double ss = 0.0;
  for (double v : values) ss += (v - mu) * (v - mu);
  return std::sqrt(ss / values.size()) / mu;
}

double serverful_cost(double total_ms, const ModelSpec& model, const ClusterSpec& cluster) {
  return (static_cast<double>(model.experts_per_layer) * model.num_layers * model.expert_mem_mb +
          cluster.m_misc_mb) * total_ms;
}

// =========================================================== baselines
std::pair<ScalingPlan, Placement> static_plan(const LoadVector& loads, const ModelSpec& model,
                                              const ClusterSpec& cluster) {
  model.validate();
  cluster.validate();
  const int n = static_cast<int>(loads.loads.size());
  if (n != model.experts_per_layer) throw std::invalid_argument("load vector does not match experts_per_layer");
  ScalingPlan plan;
  plan.layer = loads.layer;
  plan.replica_counts.assign(n, 1);
  plan.expert_mem_mb = model.expert_mem_mb;
  Placement pl;
  pl.layer = loads.layer;
  pl.per_gpu_mem_mb.assign(cluster.gpu_count, 0.0);
  for (int e = 0; e < n; ++e) {
    plan.shares.push_back({e, 0, Rational(loads.loads[e], 1)});
    const int g = e % cluster.gpu_count;  // expert e -> GPU e mod G
    pl.gpu_for.push_back({g});
    pl.per_gpu_mem_mb[g] += model.expert_mem_mb;
  }
  for (int g = 0; g < cluster.gpu_count; ++g)
    if (pl.per_gpu_mem_mb[g] > cluster.gpu_mem_capacity_mb + 1e-9)
      throw std::runtime_error("static placement does not fit GPU " + to_string(g));
  return {plan, pl};
}

LayerMetrics oracle_balance_time(const LoadVector& actual, const ClusterSpec& cluster,
                                 const ModelSpec& model) {
  cluster.validate();
  model.validate();
  // every token's work spread evenly over the GPUs: the straggler-free bound
  const double tokens = static_cast<double>(actual.total());
  LayerMetrics m;
  m.compute_ms = cluster.alpha_ms_per_token * tokens / cluster.gpu_count;
  m.comm_ms = cluster.beta_ms_per_token * tokens / cluster.gpu_count;
  m.forward_ms = m.compute_ms + 2.0 * m.comm_ms + cluster.t_misc_ms;
  m.replica_count = cluster.gpu_count;
  m.mem_mb = m.replica_count * model.expert_mem_mb;
  m.cost_mb_ms = (m.compute_ms + 2.0 * m.comm_ms) * m.mem_mb + cluster.t_misc_ms * cluster.m_misc_mb;
  return m;
}

Placement round_robin_placement(const ScalingPlan& plan, const ClusterSpec& cluster) {
  const int G = cluster.gpu_count;
  if (G < 1) throw std::invalid_argument("gpu_count must be >= 1");
  Placement pl;
  pl.layer = plan.layer;
  pl.per_gpu_mem_mb.assign(G, 0.0);
  int f = 0;  // flat replica index in (expert, ordinal) order
  for (int c : plan.replica_counts) {
    std::vector<int> gpus(std::max(c, 0));
    for (int& g : gpus) {
      g = f++ % G;
      pl.per_gpu_mem_mb[g] += plan.expert_mem_mb;
    }
    pl.gpu_for.push_back(std::move(gpus));
  }
  for (int g = 0; g < G; ++g)
    if (pl.per_gpu_mem_mb[g] > cluster.gpu_mem_capacity_mb + 1e-9)
      throw std::runtime_error("round-robin placement does not fit GPU " + to_string(g));
  return pl;
}

// ============================================================== report
double percentile(std::vector<double> values, double q) {
  if (values.empty()) throw std::invalid_argument("percentile of empty sample");
  if (q < 0.0 || q > 1.0) throw std::invalid_argument("percentile q must be in [0,1]");
  std::sort(values.begin(), values.end());
  if (q == 0.0) return values.front();
  // nearest rank: ceil(q * n), 1-based
  auto rank = static_cast<std::size_t>(std::ceil(q * static_cast<double>(values.size())));
  return values[std::max<std::size_t>(rank, 1) - 1];
}

}  // namespace moeless
