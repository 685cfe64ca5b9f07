// capi_host.cpp — the host-side entry points of the C-ABI (include/moe_b200.h)
// that need no device context: the exchange plans, and the reference planner
// restatement (scale_experts / place_experts / ReplicaRegistry / predict /
// layer_forward_time / route_tokens / popularity) plus the synthetic-input
// generators, exported so non-C++ callers and the tests reach them.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "capi_util.h"
#include "host/exchange_plan.h"
#include "kernels/dispatch_plan.h"
#include "moe_b200.h"
#include "host/moeless_api.hpp"

namespace moe {
uint64_t stream_key(uint64_t seed, uint64_t a, uint64_t b, uint64_t tag);
void synth_tokens(uint64_t key, int64_t first, int64_t tokens, int d, int E, uint16_t* x);
void synth_gate(uint64_t key, int d, int E, const double* pop, const int32_t* noise_perm, uint16_t* wg);
void synth_expert(uint64_t key, int d, int ff, uint16_t* w1, uint16_t* w3, uint16_t* w2);
}  // namespace moe

using namespace moe;

extern "C" {

int moe_exchange_plan(int G, int rank, int E, const int32_t* counts_all, const int32_t* rc, const int32_t* rg,
                      moe_chunk* sends, int* n_sends, moe_chunk* recvs, int* n_recvs, int max_chunks,
                      int64_t* rows_local, int64_t* rows_send, int64_t* seg_start, int64_t* seg_rows) {
  return guarded([&] {
    require(counts_all && rc && rg, "null argument");
    std::vector<int64_t> all(static_cast<size_t>(G) * std::max(E, 0));
    for (size_t i = 0; i < all.size(); ++i) all[i] = counts_all[i];
    HostPlan hp;
    build_exchange_plan(G, rank, E, all.data(), rc, rg, hp);
    require(static_cast<int>(hp.sends.size()) <= max_chunks && static_cast<int>(hp.recvs.size()) <= max_chunks,
            "chunk arrays too small");
    auto copy = [](const std::vector<Chunk>& v, moe_chunk* dst) {
      for (size_t i = 0; i < v.size(); ++i) dst[i] = moe_chunk{v[i].peer, v[i].replica, v[i].row_offset, v[i].rows};
    };
    if (sends) copy(hp.sends, sends);
    if (recvs) copy(hp.recvs, recvs);
    if (n_sends) *n_sends = static_cast<int>(hp.sends.size());
    if (n_recvs) *n_recvs = static_cast<int>(hp.recvs.size());
    if (rows_local) *rows_local = hp.rows_local;
    if (rows_send) *rows_send = hp.rows_send;
    for (int i = 0; i < hp.dev.R; ++i) {
      if (seg_start) seg_start[i] = hp.seg_start[i];
      if (seg_rows) seg_rows[i] = hp.rep_size[i];
    }
  });
}

int moe_exchange_plan_direct(int G, int rank, int E, const int32_t* counts_all, const int32_t* rc, const int32_t* rg,
                             int32_t* rep_target, int32_t* rep_row_base, int64_t* rows_local, int64_t* rows_send) {
  return guarded([&] {
    require(counts_all && rc && rg, "null argument");
    std::vector<int64_t> all(static_cast<size_t>(G) * std::max(E, 0));
    for (size_t i = 0; i < all.size(); ++i) all[i] = counts_all[i];
    HostPlan hp;
    build_exchange_plan(G, rank, E, all.data(), rc, rg, hp, /*direct=*/true);
    for (int f = 0; f < hp.dev.R; ++f) {
      if (rep_target) rep_target[f] = hp.dev.rep_remote[f];
      if (rep_row_base) rep_row_base[f] = hp.dev.rep_row_base[f];
    }
    if (rows_local) *rows_local = hp.rows_local;
    if (rows_send) *rows_send = hp.rows_send;
  });
}

// ------------------------------------------------------------- planner API
int moe_plan_scale(const int64_t* loads, int E, int layer, double mem, double cap, double cv, int excl,
                   int32_t* counts_out, double* alloc_out, int* steps_out, int32_t* split, double* cvt, int cap_n) {
  return guarded([&] {
    require(loads && counts_out, "null argument");
    moeless::ModelSpec m;
    m.experts_per_layer = E;
    m.top_k = 1;
    m.expert_mem_mb = mem;
    m.layer_mem_cap_mb = cap;
    moeless::ScalerConfig sc;
    sc.cv_threshold = cv;
    sc.exclude_zero_loads_from_cv = excl != 0;
    moeless::ScaleTrace tr;
    moeless::LoadVector lv{layer, std::vector<int64_t>(loads, loads + std::max(E, 0))};
    auto plan = moeless::scale_experts(lv, m, sc, &tr);
    std::copy(plan.replica_counts.begin(), plan.replica_counts.end(), counts_out);
    if (alloc_out) *alloc_out = plan.alloc_mem_mb;
    if (steps_out) *steps_out = static_cast<int>(tr.split_expert.size());
    for (int i = 0; i < cap_n && i < static_cast<int>(tr.split_expert.size()); ++i) {
      if (split) split[i] = tr.split_expert[i];
      if (cvt) cvt[i] = tr.cv[i];
    }
  });
}

struct moe_registry {
  moeless::ReplicaRegistry reg;
};

int moe_registry_create(int keep_alive, moe_registry** out) {
  return guarded([&] {
    require(out != nullptr, "null argument");
    *out = new moe_registry{moeless::ReplicaRegistry(keep_alive)};
  });
}
int moe_registry_destroy(moe_registry* r) {
  delete r;
  return MOE_OK;
}
int64_t moe_registry_size(const moe_registry* r) { return r ? static_cast<int64_t>(r->reg.size()) : -1; }

namespace {
moeless::ScalingPlan plan_of(const int64_t* loads, const int32_t* counts, int E, int layer, double mem) {
  moeless::ScalingPlan p;
  p.layer = layer;
  p.expert_mem_mb = mem;
  p.replica_counts.assign(counts, counts + E);
  int extra = 0;
  for (int e = 0; e < E; ++e) {
    extra += counts[e] - 1;
    for (int r = 0; r < counts[e]; ++r) p.shares.push_back({e, r, moeless::Rational(loads[e], counts[e])});
  }
  p.alloc_mem_mb = extra * mem;
  return p;
}
moeless::Placement placement_of(const int32_t* counts, const int32_t* gpu, int E, int G, int layer, double mem) {
  moeless::Placement p;
  p.layer = layer;
  p.per_gpu_mem_mb.assign(G, 0.0);
  int i = 0;
  for (int e = 0; e < E; ++e) {
    p.gpu_for.emplace_back();
    for (int r = 0; r < counts[e]; ++r, ++i) {
      p.gpu_for.back().push_back(gpu[i]);
      if (gpu[i] >= 0 && gpu[i] < G) p.per_gpu_mem_mb[gpu[i]] += mem;
    }
  }
  return p;
}
}  // namespace

int moe_plan_place(moe_registry* r, const int64_t* loads, const int32_t* counts, int E, int layer, double mem, int G,
                   double cap, long it, int incl, double alpha, double beta, int32_t* gpu_out, int* warm, int* cold) {
  return guarded([&] {
    require(r && loads && counts && gpu_out, "null argument");
    for (int e = 0; e < E; ++e) require(counts[e] >= 1, "replica count must be >= 1");
    auto plan = plan_of(loads, counts, E, layer, mem);
    moeless::ClusterSpec cl;
    cl.gpu_count = G;
    cl.gpu_mem_capacity_mb = cap;
    moeless::PlacerOptions opt;
    opt.load_includes_compute = incl != 0;
    opt.alpha_ms_per_token = alpha;
    opt.beta_ms_per_token = beta;
    auto res = moeless::place_experts(plan, cl, r->reg, it, opt);
    int i = 0;
    for (int e = 0; e < E; ++e)
      for (int g : res.placement.gpu_for[e]) gpu_out[i++] = g;
    if (warm) *warm = res.warm_count;
    if (cold) *cold = res.cold_count;
  });
}

int moe_registry_update(moe_registry* r, const int32_t* counts, const int32_t* gpu, int E, int G, int layer, long it) {
  return guarded([&] {
    require(r && counts && gpu, "null argument");
    moeless::update_registry(r->reg, placement_of(counts, gpu, E, G, layer, 1.0), it);
  });
}

int moe_model_forward_time(const int64_t* loads, const int32_t* counts, const int32_t* gpu, const int64_t* actual,
                           int E, int G, double alpha, double beta, double t_misc, double m_misc, double mem,
                           double* out6) {
  return guarded([&] {
    require(loads && counts && gpu && actual && out6, "null argument");
    auto plan = plan_of(loads, counts, E, 0, mem);
    auto pl = placement_of(counts, gpu, E, G, 0, mem);
    moeless::ClusterSpec cl;
    cl.gpu_count = G;
    cl.alpha_ms_per_token = alpha;
    cl.beta_ms_per_token = beta;
    cl.t_misc_ms = t_misc;
    cl.m_misc_mb = m_misc;
    moeless::ModelSpec ms;
    ms.experts_per_layer = E;
    ms.expert_mem_mb = mem;
    auto m = moeless::layer_forward_time(plan, pl, moeless::LoadVector{0, std::vector<int64_t>(actual, actual + E)}, cl,
                                         ms);
    out6[0] = m.compute_ms;
    out6[1] = m.comm_ms;
    out6[2] = m.forward_ms;
    out6[3] = m.replica_count;
    out6[4] = m.mem_mb;
    out6[5] = m.cost_mb_ms;
  });
}

int moe_plan_predict(int kind, const int64_t* actual, int E, int layer, const int64_t* history, int hlen,
                     const double* acc, int L, int distance, double decay, int window, long it, uint64_t seed,
                     const double* pop, int64_t* out, int* fallback) {
  return guarded([&] {
    require(actual && out, "null argument");
    require(kind >= 0 && kind <= 2, "unknown predictor kind");
    moeless::PredictorProfile p;
    p.kind = static_cast<moeless::PredictorKind>(kind);
    p.distance = distance;
    p.distance_decay = decay;
    p.history_window = window;
    if (acc) p.per_layer_accuracy.assign(acc, acc + L);
    std::vector<moeless::LoadVector> hist;
    for (int i = 0; i < hlen; ++i)
      hist.push_back({layer, std::vector<int64_t>(history + static_cast<size_t>(i) * E, history + static_cast<size_t>(i + 1) * E)});
    std::vector<double> pw;
    if (pop) pw.assign(pop, pop + E);
    bool fb = false;
    auto r = moeless::predict({layer, std::vector<int64_t>(actual, actual + E)}, hist, p, it, seed, pw, &fb);
    std::copy(r.loads.begin(), r.loads.end(), out);
    if (fallback) *fallback = fb ? 1 : 0;
  });
}

double moe_measure_accuracy(const int64_t* pred, const int64_t* actual, int E) {
  double v = -1.0;
  int rc = guarded([&] {
    v = moeless::measure_accuracy({0, std::vector<int64_t>(pred, pred + E)}, {0, std::vector<int64_t>(actual, actual + E)});
  });
  return rc == MOE_OK ? v : -1.0;
}

double moe_percentile(const double* v, int n, double q) {
  double out = -1.0;
  int rc = guarded([&] { out = moeless::percentile(std::vector<double>(v, v + std::max(n, 0)), q); });
  return rc == MOE_OK ? out : -1.0;
}

int moe_route_tokens(int64_t T, int layer, long it, int E, int L, double s, uint64_t seed, int k, int drift,
                     int64_t* loads) {
  return guarded([&] {
    require(loads != nullptr, "null argument");
    auto prof = moeless::make_popularity_profile(E, L, s, seed, false, drift);
    moeless::IterationBatch b;
    b.iteration = it;
    b.token_count = T;
    auto lv = moeless::route_tokens(b, layer, prof, k, E, seed);
    std::copy(lv.loads.begin(), lv.loads.end(), loads);
  });
}

int moe_popularity(int E, int L, double s, uint64_t seed, int layer, long it, int drift, int32_t* perm, double* w) {
  return guarded([&] {
    auto prof = moeless::make_popularity_profile(E, L, s, seed, false, drift);
    auto p = moeless::effective_permutation(prof, layer, it);
    if (perm) std::copy(p.begin(), p.end(), perm);
    if (w) {
      auto ww = moeless::popularity_weights(prof, layer, it, moeless::Phase::prefill);
      std::copy(ww.begin(), ww.end(), w);
    }
  });
}

uint64_t moe_stream_key(uint64_t seed, uint64_t a, uint64_t b, uint64_t tag) { return stream_key(seed, a, b, tag); }

int moe_synth_tokens(uint64_t key, int64_t first, int64_t T, int d, int E, uint16_t* x) {
  return guarded([&] {
    require(x && T >= 0 && d > E && E >= 1, "bad synth_tokens arguments");
    synth_tokens(key, first, T, d, E, x);
  });
}

int moe_synth_gate(uint64_t key, int d, int E, const double* pop, const int32_t* noise_perm, uint16_t* wg) {
  return guarded([&] {
    require(pop && noise_perm && wg && d > E, "bad synth_gate arguments");
    synth_gate(key, d, E, pop, noise_perm, wg);
  });
}

int moe_synth_expert(uint64_t key, int d, int ff, uint16_t* w1, uint16_t* w3, uint16_t* w2) {
  return guarded([&] {
    require(w1 && w3 && w2, "null argument");
    synth_expert(key, d, ff, w1, w3, w2);
  });
}

// ------------------------------------------------ baselines / cost model rows
int moe_static_plan(const int64_t* loads, int E, int G, double mem, double gpu_mem, int32_t* gpu_out) {
  return guarded([&] {
    require(loads && gpu_out, "null argument");
    moeless::ModelSpec ms;
    ms.experts_per_layer = E;
    ms.expert_mem_mb = mem;
    moeless::ClusterSpec cl;
    cl.gpu_count = G;
    cl.gpu_mem_capacity_mb = gpu_mem;
    auto sp = moeless::static_plan(moeless::LoadVector{0, std::vector<int64_t>(loads, loads + E)}, ms, cl);
    for (int e = 0; e < E; ++e) gpu_out[e] = sp.second.gpu_for[e][0];
  });
}

int moe_round_robin_placement(const int32_t* counts, int E, int G, double mem, double gpu_mem, int32_t* gpu_out) {
  return guarded([&] {
    require(counts && gpu_out, "null argument");
    moeless::ScalingPlan plan;
    plan.replica_counts.assign(counts, counts + E);
    plan.expert_mem_mb = mem;
    moeless::ClusterSpec cl;
    cl.gpu_count = G;
    cl.gpu_mem_capacity_mb = gpu_mem;
    auto pl = moeless::round_robin_placement(plan, cl);
    int i = 0;
    for (const auto& v : pl.gpu_for)
      for (int g : v) gpu_out[i++] = g;
  });
}

int moe_gpu_comm_times(const int64_t* loads, const int32_t* counts, const int32_t* gpu, int E, int G, double beta,
                       double* out) {
  return guarded([&] {
    require(loads && counts && gpu && out, "null argument");
    auto v = moeless::gpu_comm_times(plan_of(loads, counts, E, 0, 0.0), placement_of(counts, gpu, E, G, 0, 0.0), beta);
    std::copy(v.begin(), v.end(), out);
  });
}

int moe_oracle_balance_time(const int64_t* actual, int E, int G, double alpha, double beta, double t_misc,
                            double m_misc, double mem, double* out6) {
  return guarded([&] {
    require(actual && out6, "null argument");
    moeless::ClusterSpec cl;
    cl.gpu_count = G;
    cl.alpha_ms_per_token = alpha;
    cl.beta_ms_per_token = beta;
    cl.t_misc_ms = t_misc;
    cl.m_misc_mb = m_misc;
    moeless::ModelSpec ms;
    ms.experts_per_layer = E;
    ms.expert_mem_mb = mem;
    auto m = moeless::oracle_balance_time(moeless::LoadVector{0, std::vector<int64_t>(actual, actual + E)}, cl, ms);
    const double v[6] = {m.compute_ms, m.comm_ms, m.forward_ms, static_cast<double>(m.replica_count), m.mem_mb,
                         m.cost_mb_ms};
    std::copy(v, v + 6, out6);
  });
}

int moe_verify_plan(const int64_t* loads, int E, const int32_t* counts, int n_counts, const int32_t* share_expert,
                    const int32_t* share_ordinal, const int64_t* share_num, const int64_t* share_den, int n_shares,
                    double alloc_mem_mb, double mem, double layer_cap_mb, double cv_threshold, int exclude_zero,
                    int* ok, char* issues, int cap) {
  return guarded([&] {
    require(loads && ok && (n_counts == 0 || counts), "null argument");
    moeless::ScalingPlan plan;
    plan.replica_counts.assign(counts, counts + n_counts);
    for (int i = 0; i < n_shares; ++i)
      plan.shares.push_back({share_expert[i], share_ordinal[i], moeless::Rational(share_num[i], share_den[i])});
    plan.alloc_mem_mb = alloc_mem_mb;
    plan.expert_mem_mb = mem;
    moeless::ModelSpec ms;
    ms.experts_per_layer = E;
    ms.expert_mem_mb = mem;
    ms.layer_mem_cap_mb = layer_cap_mb;
    moeless::ScalerConfig sc;
    sc.cv_threshold = cv_threshold;
    sc.exclude_zero_loads_from_cv = exclude_zero != 0;
    auto rep = moeless::verify_plan(plan, moeless::LoadVector{0, std::vector<int64_t>(loads, loads + E)}, ms, sc);
    *ok = rep.ok ? 1 : 0;
    std::string all;
    for (const auto& m : rep.issues) all += m + "\n";
    if (issues && cap > 0) {
      const size_t n = std::min(all.size(), static_cast<size_t>(cap - 1));
      std::memcpy(issues, all.data(), n);
      issues[n] = 0;
    }
  });
}

int moe_apply_finetuning(double* accuracy, int n, double threshold, int32_t* fine_tuned) {
  return guarded([&] {
    require(accuracy && fine_tuned, "null argument");
    moeless::PredictorProfile p;
    p.kind = moeless::PredictorKind::noisy;
    p.per_layer_accuracy.assign(accuracy, accuracy + n);
    p.accuracy_threshold = threshold;
    moeless::apply_layer_aware_finetuning(p);
    for (int l = 0; l < n; ++l) {
      accuracy[l] = p.per_layer_accuracy[l];
      fine_tuned[l] = p.fine_tuned[l] ? 1 : 0;
    }
  });
}

double moe_coefficient_of_variation(const double* values, int n) {
  double r = -1.0;
  const int rc = guarded([&] { r = moeless::coefficient_of_variation(std::vector<double>(values, values + n)); });
  return rc == MOE_OK ? r : -1.0;
}

double moe_serverful_cost(double total_ms, int num_layers, int E, double mem, double m_misc) {
  moeless::ModelSpec ms;
  ms.num_layers = num_layers;
  ms.experts_per_layer = E;
  ms.expert_mem_mb = mem;
  moeless::ClusterSpec cl;
  cl.m_misc_mb = m_misc;
  return moeless::serverful_cost(total_ms, ms, cl);
}

}  // extern "C"
