// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference simulator sources
// (/root/reference/proj/src/*.cpp), compiled by oracle/Makefile into
// oracle/_ref/libmoeless_ref.so.  Python tests and the bench's cpu_baseline /
// `--impl reference` leg load it with ctypes so that every planner decision
// and every load histogram the product computes can be compared with what the
// reference itself computes on identical inputs.
//
// Each wrapper names the reference entry point it forwards to.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include <algorithm>

#include "moeless/baselines.hpp"
#include "moeless/config.hpp"
#include "moeless/simulator.hpp"
#include "moeless/cost_model.hpp"
#include "moeless/placer.hpp"
#include "moeless/predictor.hpp"
#include "moeless/report.hpp"
#include "moeless/scaler.hpp"
#include "moeless/workload.hpp"

using namespace moeless;

namespace {
thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  return dynamic_cast<const std::invalid_argument*>(&e) ? 1 : 2;
}

LoadVector lv(const std::int64_t* v, int n, int layer = 0) {
  LoadVector out;
  out.layer = layer;
  out.loads.assign(v, v + n);
  return out;
}

ScalingPlan plan_from(const std::int64_t* loads, const int* counts, int experts, int layer,
                      double expert_mem_mb) {
  ScalingPlan plan;
  plan.layer = layer;
  plan.replica_counts.assign(counts, counts + experts);
  plan.expert_mem_mb = expert_mem_mb;
  int extra = 0;
  for (int e = 0; e < experts; ++e) {
    extra += counts[e] - 1;
    for (int r = 0; r < counts[e]; ++r) plan.shares.push_back({e, r, Rational(loads[e], counts[e])});
  }
  plan.alloc_mem_mb = extra * expert_mem_mb;
  return plan;
}

Placement placement_from(const int* counts, const int* gpu_flat, int experts, int gpus,
                         int layer, double expert_mem_mb) {
  Placement p;
  p.layer = layer;
  p.gpu_for.resize(experts);
  p.per_gpu_mem_mb.assign(gpus, 0.0);
  int idx = 0;
  for (int e = 0; e < experts; ++e)
    for (int r = 0; r < counts[e]; ++r, ++idx) {
      p.gpu_for[e].push_back(gpu_flat[idx]);
      if (gpu_flat[idx] >= 0 && gpu_flat[idx] < gpus) p.per_gpu_mem_mb[gpu_flat[idx]] += expert_mem_mb;
    }
  return p;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// make_popularity_profile + effective_permutation (workload.cpp:30-75)
int ref_popularity_perm(int experts, int layers, double s, std::uint64_t seed, int layer,
                        long iteration, int drift_period, int* perm_out, double* weights_out) {
  try {
    auto prof = make_popularity_profile(experts, layers, s, seed, false, drift_period);
    auto perm = effective_permutation(prof, layer, iteration);
    std::memcpy(perm_out, perm.data(), sizeof(int) * experts);
    if (weights_out) {
      auto w = popularity_weights(prof, layer, iteration, Phase::prefill);
      std::memcpy(weights_out, w.data(), sizeof(double) * experts);
    }
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

// route_tokens (workload.cpp:188-230)
int ref_route_tokens(std::int64_t tokens, int layer, long iteration, int experts, int layers,
                     double s, std::uint64_t seed, int top_k, int drift_period,
                     std::int64_t* loads_out) {
  try {
    auto prof = make_popularity_profile(experts, layers, s, seed, false, drift_period);
    IterationBatch b;
    b.iteration = iteration;
    b.token_count = tokens;
    auto out = route_tokens(b, layer, prof, top_k, experts, seed);
    std::memcpy(loads_out, out.loads.data(), sizeof(std::int64_t) * experts);
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

// scale_experts + verify_plan (scaler.cpp:55-173)
int ref_scale_experts(const std::int64_t* loads, int experts, int layer, double expert_mem_mb,
                      double layer_mem_cap_mb, double cv_threshold, int exclude_zero,
                      int* counts_out, double* alloc_out, int* steps_out, int* split_out,
                      int split_cap, double* cv_out, int* verify_ok) {
  try {
    ModelSpec m;
    m.experts_per_layer = experts;
    m.top_k = 1;
    m.expert_mem_mb = expert_mem_mb;
    m.layer_mem_cap_mb = layer_mem_cap_mb;
    ScalerConfig cfg;
    cfg.cv_threshold = cv_threshold;
    cfg.exclude_zero_loads_from_cv = exclude_zero != 0;
    ScaleTrace tr;
    auto in = lv(loads, experts, layer);
    auto plan = scale_experts(in, m, cfg, &tr);
    std::memcpy(counts_out, plan.replica_counts.data(), sizeof(int) * experts);
    if (alloc_out) *alloc_out = plan.alloc_mem_mb;
    if (steps_out) *steps_out = static_cast<int>(tr.split_expert.size());
    for (int i = 0; split_out && i < split_cap && i < (int)tr.split_expert.size(); ++i) {
      split_out[i] = tr.split_expert[i];
      if (cv_out) cv_out[i] = tr.cv[i];
    }
    if (verify_ok) *verify_ok = verify_plan(plan, in, m, cfg).ok ? 1 : 0;
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

// ReplicaRegistry (placer.cpp:11-43) as an opaque handle
void* ref_registry_new(int keep_alive) {
  try { return new ReplicaRegistry(keep_alive); } catch (const std::exception& e) { fail(e); return nullptr; }
}
void ref_registry_free(void* h) { delete static_cast<ReplicaRegistry*>(h); }
long ref_registry_size(void* h) { return (long)static_cast<ReplicaRegistry*>(h)->size(); }

// place_experts (placer.cpp:45-122)
int ref_place_experts(void* reg, const std::int64_t* plan_loads, const int* counts, int experts,
                      int layer, double expert_mem_mb, int gpus, double gpu_mem_mb, long iteration,
                      int include_compute, double alpha, double beta, int* gpu_out, int* warm,
                      int* cold) {
  try {
    auto plan = plan_from(plan_loads, counts, experts, layer, expert_mem_mb);
    ClusterSpec c;
    c.gpu_count = gpus;
    c.gpu_mem_capacity_mb = gpu_mem_mb;
    PlacerOptions opt;
    opt.load_includes_compute = include_compute != 0;
    opt.alpha_ms_per_token = alpha;
    opt.beta_ms_per_token = beta;
    auto res = place_experts(plan, c, *static_cast<ReplicaRegistry*>(reg), iteration, opt);
    int idx = 0;
    for (int e = 0; e < experts; ++e)
      for (int r = 0; r < counts[e]; ++r) gpu_out[idx++] = res.placement.gpu_for[e][r];
    *warm = res.warm_count;
    *cold = res.cold_count;
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

// update_registry (placer.cpp:124-130)
int ref_update_registry(void* reg, const int* counts, const int* gpu_flat, int experts, int gpus,
                        int layer, long iteration) {
  try {
    auto p = placement_from(counts, gpu_flat, experts, gpus, layer, 1.0);
    update_registry(*static_cast<ReplicaRegistry*>(reg), p, iteration);
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

// layer_forward_time (cost_model.cpp:91-122); out = compute, comm, forward, replicas, mem, cost
int ref_layer_forward_time(const std::int64_t* plan_loads, const int* counts, const int* gpu_flat,
                           const std::int64_t* actual, int experts, int gpus, double alpha,
                           double beta, double t_misc, double m_misc, double expert_mem_mb,
                           double* out6) {
  try {
    auto plan = plan_from(plan_loads, counts, experts, 0, expert_mem_mb);
    auto p = placement_from(counts, gpu_flat, experts, gpus, 0, expert_mem_mb);
    ClusterSpec c;
    c.gpu_count = gpus;
    c.alpha_ms_per_token = alpha;
    c.beta_ms_per_token = beta;
    c.t_misc_ms = t_misc;
    c.m_misc_mb = m_misc;
    ModelSpec m;
    m.experts_per_layer = experts;
    m.expert_mem_mb = expert_mem_mb;
    auto r = layer_forward_time(plan, p, lv(actual, experts), c, m);
    out6[0] = r.compute_ms;
    out6[1] = r.comm_ms;
    out6[2] = r.forward_ms;
    out6[3] = r.replica_count;
    out6[4] = r.mem_mb;
    out6[5] = r.cost_mb_ms;
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

// predict (predictor.cpp:146-166). kind: 0 oracle, 1 noisy, 2 historical
int ref_predict(int kind, const std::int64_t* actual, int experts, int layer,
                const std::int64_t* history, int history_len, const double* accuracy,
                int num_layers, int distance, double decay, int window, long iteration,
                std::uint64_t seed, const double* popularity, std::int64_t* out, int* fallback) {
  try {
    PredictorProfile p;
    p.kind = static_cast<PredictorKind>(kind);
    p.distance = distance;
    p.distance_decay = decay;
    p.history_window = window;
    if (accuracy) p.per_layer_accuracy.assign(accuracy, accuracy + num_layers);
    std::vector<LoadVector> hist;
    for (int i = 0; i < history_len; ++i) hist.push_back(lv(history + (long)i * experts, experts, layer));
    std::vector<double> pop;
    if (popularity) pop.assign(popularity, popularity + experts);
    bool fb = false;
    auto r = predict(lv(actual, experts, layer), hist, p, iteration, seed, pop, &fb);
    std::memcpy(out, r.loads.data(), sizeof(std::int64_t) * experts);
    if (fallback) *fallback = fb ? 1 : 0;
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

// measure_accuracy (predictor.cpp:168-186)
double ref_measure_accuracy(const std::int64_t* pred, const std::int64_t* actual, int experts) {
  try { return measure_accuracy(lv(pred, experts), lv(actual, experts)); } catch (const std::exception& e) { fail(e); return -1.0; }
}

// percentile (report.cpp:150-159)
double ref_percentile(const double* v, int n, double q) {
  try { return percentile(std::vector<double>(v, v + n), q); } catch (const std::exception& e) { fail(e); return -1.0; }
}

// static_plan (baselines.cpp:32-60) placement only
int ref_static_plan(const std::int64_t* loads, int experts, int gpus, double expert_mem_mb,
                    double gpu_mem_mb, int* gpu_out) {
  try {
    ModelSpec m;
    m.experts_per_layer = experts;
    m.expert_mem_mb = expert_mem_mb;
    ClusterSpec c;
    c.gpu_count = gpus;
    c.gpu_mem_capacity_mb = gpu_mem_mb;
    auto r = static_plan(lv(loads, experts), m, c);
    for (int e = 0; e < experts; ++e) gpu_out[e] = r.second.gpu_for[e][0];
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

// gpu_comm_times (cost_model.cpp:67-89)
int ref_gpu_comm_times(const std::int64_t* plan_loads, const int* counts, const int* gpu_flat, int experts,
                       int gpus, double beta, double* out) {
  try {
    auto v = gpu_comm_times(plan_from(plan_loads, counts, experts, 0, 0.0),
                            placement_from(counts, gpu_flat, experts, gpus, 0, 0.0), beta);
    std::memcpy(out, v.data(), sizeof(double) * v.size());
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

// oracle_balance_time (baselines.cpp:141-154)
int ref_oracle_balance_time(const std::int64_t* actual, int experts, int gpus, double alpha, double beta,
                            double t_misc, double m_misc, double expert_mem_mb, double* out6) {
  try {
    ClusterSpec c;
    c.gpu_count = gpus;
    c.alpha_ms_per_token = alpha;
    c.beta_ms_per_token = beta;
    c.t_misc_ms = t_misc;
    c.m_misc_mb = m_misc;
    ModelSpec m;
    m.experts_per_layer = experts;
    m.expert_mem_mb = expert_mem_mb;
    auto r = oracle_balance_time(lv(actual, experts), c, m);
    const double v[6] = {r.compute_ms, r.comm_ms, r.forward_ms, (double)r.replica_count, r.mem_mb, r.cost_mb_ms};
    std::memcpy(out6, v, sizeof v);
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

// verify_plan (scaler.cpp:99-173) on an explicit (possibly broken) plan
int ref_verify_plan(const std::int64_t* loads, int experts, const int* counts, int n_counts, const int* s_expert,
                    const int* s_ordinal, const std::int64_t* s_num, const std::int64_t* s_den, int n_shares,
                    double alloc_mem_mb, double expert_mem_mb, double cap_mb, double cv_threshold,
                    int exclude_zero, int* ok, char* issues, int cap) {
  try {
    ScalingPlan plan;
    plan.replica_counts.assign(counts, counts + n_counts);
    for (int i = 0; i < n_shares; ++i) plan.shares.push_back({s_expert[i], s_ordinal[i], Rational(s_num[i], s_den[i])});
    plan.alloc_mem_mb = alloc_mem_mb;
    plan.expert_mem_mb = expert_mem_mb;
    ModelSpec m;
    m.experts_per_layer = experts;
    m.expert_mem_mb = expert_mem_mb;
    m.layer_mem_cap_mb = cap_mb;
    ScalerConfig cfg;
    cfg.cv_threshold = cv_threshold;
    cfg.exclude_zero_loads_from_cv = exclude_zero != 0;
    auto rep = verify_plan(plan, lv(loads, experts), m, cfg);
    *ok = rep.ok ? 1 : 0;
    std::string all;
    for (const auto& x : rep.issues) all += x + "\n";
    const std::size_t n = std::min(all.size(), static_cast<std::size_t>(cap - 1));
    std::memcpy(issues, all.data(), n);
    issues[n] = 0;
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

// apply_layer_aware_finetuning (predictor.cpp:188-199)
int ref_apply_finetuning(double* acc, int n, double threshold, int* fine_tuned) {
  try {
    PredictorProfile p;
    p.kind = PredictorKind::noisy;
    p.per_layer_accuracy.assign(acc, acc + n);
    p.accuracy_threshold = threshold;
    apply_layer_aware_finetuning(p);
    for (int l = 0; l < n; ++l) {
      acc[l] = p.per_layer_accuracy[l];
      fine_tuned[l] = p.fine_tuned[l] ? 1 : 0;
    }
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

// coefficient_of_variation / serverful_cost (cost_model.cpp:124-139)
double ref_coefficient_of_variation(const double* v, int n) {
  try { return coefficient_of_variation(std::vector<double>(v, v + n)); } catch (const std::exception& e) { fail(e); return -1.0; }
}
double ref_serverful_cost(double total_ms, int layers, int experts, double expert_mem_mb, double m_misc) {
  ModelSpec m;
  m.num_layers = layers;
  m.experts_per_layer = experts;
  m.expert_mem_mb = expert_mem_mb;
  ClusterSpec c;
  c.m_misc_mb = m_misc;
  return serverful_cost(total_ms, m, c);
}

// The reference simulator end to end (config.cpp:90 parse_config_text ->
// workload.cpp:90 parse_trace -> simulator.cpp:71 run -> report.cpp:48
// summary_json), for driving it with B200-calibrated alpha/beta/t_misc.
// Writes the summary JSON into out (NUL-terminated, truncated to cap).
int ref_simulate(const char* config_text, const char* trace_path, char* out, int cap) {
  try {
    SimConfig cfg = parse_config_text(config_text, "<calibrated>");
    auto trace = parse_trace(trace_path);
    auto rep = run(cfg, trace);
    const std::string js = summary_json(rep);
    const int n = std::min<int>(cap - 1, static_cast<int>(js.size()));
    std::memcpy(out, js.data(), n);
    out[n] = 0;
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

// parse_trace + batch_requests (workload.cpp:90-186): writes up to cap
// (iteration, phase 0/1, token_count) triples, returns the batch count.
long ref_batch_trace(const char* trace_path, long* out, long cap) {
  try {
    auto b = batch_requests(parse_trace(trace_path));
    for (long i = 0; i < static_cast<long>(b.size()) && i < cap; ++i) {
      out[3 * i] = b[i].iteration;
      out[3 * i + 1] = b[i].phase == Phase::decode ? 1 : 0;
      out[3 * i + 2] = static_cast<long>(b[i].token_count);
    }
    return static_cast<long>(b.size());
  } catch (const std::exception& e) { fail(e); return -1; }
}

// The reference's per-layer CPU path, exactly as run() sequences it
// (simulator.cpp:116-201): route_tokens -> predict -> scale_experts ->
// place_experts -> layer_forward_time -> update_registry.  Runs `iters`
// iterations of one layer and returns the wall seconds spent.
double ref_cpu_layer_path(std::int64_t tokens, int experts, int top_k, double s, std::uint64_t seed,
                          int gpus, double expert_mem_mb, double layer_mem_cap_mb, int iters,
                          std::int64_t* last_loads) {
  try {
    auto prof = make_popularity_profile(experts, 2, s, seed);
    ModelSpec m;
    m.num_layers = 2;
    m.experts_per_layer = experts;
    m.top_k = top_k;
    m.expert_mem_mb = expert_mem_mb;
    m.layer_mem_cap_mb = layer_mem_cap_mb;
    ClusterSpec c;
    c.gpu_count = gpus;
    c.gpu_mem_capacity_mb = 180000.0;
    PredictorProfile pp;
    pp.kind = PredictorKind::oracle;
    pp.per_layer_accuracy = {1.0, 1.0};
    ReplicaRegistry reg(50);
    std::vector<LoadVector> hist;
    double sink = 0.0;
    const auto t0 = std::chrono::steady_clock::now();
    for (int it = 0; it < iters; ++it) {
      IterationBatch b;
      b.iteration = it;
      b.token_count = tokens;
      auto actual = route_tokens(b, 1, prof, top_k, experts, seed);
      auto pred = predict(actual, hist, pp, it, seed);
      auto plan = scale_experts(pred, m, {});
      auto placed = place_experts(plan, c, reg, it);
      auto lm = layer_forward_time(plan, placed.placement, actual, c, m);
      update_registry(reg, placed.placement, it);
      sink += lm.forward_ms;
      if (it == iters - 1 && last_loads)
        std::memcpy(last_loads, actual.loads.data(), sizeof(std::int64_t) * experts);
    }
    const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return sink >= 0 ? dt : -dt;
  } catch (const std::exception& e) { fail(e); return -1.0; }
}

}  // extern "C"
