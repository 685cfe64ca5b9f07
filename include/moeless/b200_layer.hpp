// moeless/b200_layer.hpp — header-only C++ binding of the B200 MoE layer
// (C-ABI include/moe_b200.h) for code written against the REFERENCE's C++
// API (proj/include/moeless/*.hpp).
//
// It includes the reference's own headers ("moeless/types.hpp",
// "moeless/placer.hpp") from the caller's include path — this repository
// ships no header of those names — and uses only their public members:
// ModelSpec, ClusterSpec, LoadVector, ScalingPlan, Placement, LayerMetrics
// (types.hpp:16-80, placer.hpp:15-21).  Status codes come back as the
// exceptions the reference throws (std::invalid_argument for bad input,
// std::runtime_error otherwise, placer.cpp:101-104 wording kept by the C-ABI).
//
// Drop-in at the reference's call site, proj/src/simulator.cpp:193-194:
//
//   const LayerMetrics m =
//       layer_forward_time(plan, placement, actual[l], config.cluster, config.model);
// becomes
//   const LayerMetrics m =
//       b200::layer_forward_time(plan, placement, actual[l], config.cluster, config.model);
//
// with this header force-included (g++ -include moeless/b200_layer.hpp) and
// the program linked against libmoe_b200.so + libcudart.  Same signature,
// same LayerMetrics fields — but compute/comm/forward are MEASURED on the
// GPU: the real layer (dispatch -> tcgen05 SwiGLU grouped GEMM -> combine,
// expert-parallel over cluster.gpu_count ranks) runs the plan and placement
// the reference's planner chose on tokens routed exactly as `actual` says
// (moe_layer_forward_ids: the reference's route_tokens histogram IS the
// routing; the gate is not needed).  INTEGRATION.md §1 has the recipe and
// tests/test_dropin.py builds and runs it.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "moe_b200.h"
#include "moeless/placer.hpp"
#include "moeless/types.hpp"

namespace moeless::b200 {

inline void check(int rc) {
  if (rc == MOE_OK) return;
  const std::string msg = moe_last_error();
  if (rc == MOE_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// ScalingPlan.replica_counts (types.hpp:59) / Placement.gpu_for (placer.hpp:17)
// flattened into the C-ABI replica table.
inline void flatten(const ScalingPlan& plan, const Placement& placement, std::vector<int32_t>& rc,
                    std::vector<int32_t>& rg) {
  rc.assign(plan.replica_counts.begin(), plan.replica_counts.end());
  rg.clear();
  for (const auto& per : placement.gpu_for) rg.insert(rg.end(), per.begin(), per.end());
}

// Per-token routing whose histogram is exactly `loads` (sum = T * k, every
// load <= T): the experts, each repeated loads[e] times in expert order, are
// dealt column-major — token t takes positions t, t + T, ..., t + (k-1) T.
// Two positions of one expert are < T apart, so a token never gets an
// expert twice (route_tokens' without-replacement rule, workload.cpp:221-226).
inline std::vector<int32_t> ids_for_loads(const std::vector<std::int64_t>& loads, int k, int64_t* tokens_out) {
  std::int64_t total = 0;
  for (auto v : loads) {
    if (v < 0) throw std::invalid_argument("negative actual load");
    total += v;
  }
  if (k < 1 || total % k != 0) throw std::invalid_argument("actual loads do not sum to tokens * top_k");
  const std::int64_t T = total / k;
  for (auto v : loads)
    if (v > T) throw std::invalid_argument("an expert has more loads than tokens");
  std::vector<int32_t> seq;
  seq.reserve(static_cast<size_t>(total));
  for (size_t e = 0; e < loads.size(); ++e) seq.insert(seq.end(), static_cast<size_t>(loads[e]), static_cast<int32_t>(e));
  std::vector<int32_t> ids(static_cast<size_t>(total));
  for (std::int64_t t = 0; t < T; ++t)
    for (int j = 0; j < k; ++j) ids[static_cast<size_t>(t * k + j)] = seq[static_cast<size_t>(t + j * T)];
  *tokens_out = T;
  return ids;
}

// One rank of an MoE layer stack (one moe_ctx).
class Layer {
 public:
  // `model.num_layers`, `experts_per_layer`, `top_k`, `expert_mem_mb`,
  // `layer_mem_cap_mb` come from the reference ModelSpec.
  Layer(const ModelSpec& model, int d_model, int d_ff, int max_tokens, int world_size = 1, int rank = 0,
        int device = 0, int exchange_mode = MOE_EXCHANGE_P2P, const void* nccl_unique_id = nullptr,
        double gpu_mem_capacity_mb = 180000.0) {
    moe_ctx_desc d{};
    d.num_layers = model.num_layers;
    d.num_experts = model.experts_per_layer;
    d.top_k = model.top_k;
    d.d_model = d_model;
    d.d_ff = d_ff;
    d.max_tokens = max_tokens;
    d.world_size = world_size;
    d.rank = rank;
    d.device = device;
    d.exchange_mode = exchange_mode;
    d.nccl_unique_id = nccl_unique_id;
    d.expert_mem_mb = model.expert_mem_mb;
    d.layer_mem_cap_mb = model.layer_mem_cap_mb;
    d.gpu_mem_capacity_mb = gpu_mem_capacity_mb;
    d.cv_threshold = 0.2;
    d.keep_alive_iters = 50;
    check(moe_ctx_create(&d, &ctx_));
    E_ = model.experts_per_layer;
  }
  ~Layer() {
    if (ctx_) moe_ctx_destroy(ctx_);
  }
  Layer(const Layer&) = delete;
  Layer& operator=(const Layer&) = delete;

  void load_expert(int layer, int expert, const uint16_t* w1, const uint16_t* w3, const uint16_t* w2) {
    check(moe_load_expert_weights(ctx_, layer, expert, w1, w3, w2));
  }
  void set_gate(int layer, const uint16_t* wg) { check(moe_set_gate_weights(ctx_, layer, wg)); }
  void set_placement(const ScalingPlan& plan, const Placement& placement) {
    std::vector<int32_t> rc, rg;
    flatten(plan, placement, rc, rg);
    check(moe_set_placement(ctx_, plan.layer, rc.data(), rg.data()));
  }
  // The layer for a (plan, placement) pair, routed by the gate (device buffers).
  moe_layer_stats forward(const ScalingPlan& plan, const Placement& placement, const uint16_t* x_dev, int tokens,
                          uint16_t* y_dev, long iteration, void* stream = nullptr) {
    set_placement(plan, placement);
    moe_layer_stats st{};
    check(moe_layer_forward(ctx_, plan.layer, x_dev, tokens, y_dev, MOE_PLAN_FIXED, iteration, &st, stream));
    return st;
  }
  // Same, routed by caller-given ids [tokens, k] (device; weights NULL = 1/k).
  moe_layer_stats forward_ids(int layer, const uint16_t* x_dev, const int32_t* ids_dev, const float* w_dev,
                              int tokens, uint16_t* y_dev, long iteration, void* stream = nullptr) {
    moe_layer_stats st{};
    check(moe_layer_forward_ids(ctx_, layer, x_dev, ids_dev, w_dev, tokens, y_dev, MOE_PLAN_FIXED, iteration, &st,
                                stream));
    return st;
  }
  moe_ctx* handle() const { return ctx_; }

 private:
  moe_ctx* ctx_ = nullptr;
  int E_ = 0;
};

// The GPU side of b200::layer_forward_time: cluster.gpu_count ranks (one
// moe_ctx each, peer-memory expert parallelism; rank r on device r mod the
// visible devices, so a one-GPU box runs every rank on the same B200),
// synthetic bf16 expert weights keyed per (seed, layer, expert) and tokens
// keyed per call.  d_model / d_ff are not part of the reference ModelSpec:
// env MOE_B200_D_MODEL / MOE_B200_D_FF (default 1024 / 3584, BASELINE cfg1).
class Engine {
 public:
  Engine(const ClusterSpec& cluster, const ModelSpec& model) : model_(model) {
    d_ = env_int("MOE_B200_D_MODEL", 1024);
    ff_ = env_int("MOE_B200_D_FF", 3584);
    seed_ = static_cast<uint64_t>(env_int("MOE_B200_SEED", 1));
    G_ = cluster.gpu_count;
    int ndev = 0;
    cuda_check(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
    if (ndev < 1) throw std::runtime_error("no CUDA device");
    for (int r = 0; r < G_; ++r) dev_.push_back(r % ndev);
  }

  LayerMetrics forward(const ScalingPlan& plan, const Placement& placement, const LoadVector& actual,
                       const ClusterSpec& cluster, const ModelSpec& model) {
    if (cluster.gpu_count != G_ || model.experts_per_layer != model_.experts_per_layer)
      throw std::invalid_argument("cluster or model changed between calls on one thread");
    const int E = model.experts_per_layer, k = model.top_k, layer = plan.layer;
    if (static_cast<int>(actual.loads.size()) != E)
      throw std::invalid_argument("actual load vector does not match plan expert count");
    std::int64_t T = 0;
    const std::vector<int32_t> ids = ids_for_loads(actual.loads, k, &T);
    ensure(static_cast<int>(T), layer);
    std::vector<int32_t> rc, rg;
    flatten(plan, placement, rc, rg);
    // tokens of this call, sharded contiguously over the ranks (data parallel)
    const uint64_t key = moe_stream_key(seed_, static_cast<uint64_t>(layer), calls_++, 0x78746F6Bull);
    std::vector<moe_layer_stats> st(G_);
    std::vector<std::string> err(G_);
    auto run_rank = [&](int r) {
      try {
        const int64_t t0 = T * r / G_, t1 = T * (r + 1) / G_, n = t1 - t0;
        Rank& R = ranks_[r];
        cuda_check(cudaSetDevice(dev_[r]), "cudaSetDevice");
        std::vector<uint16_t> xh(static_cast<size_t>(std::max<int64_t>(n, 1)) * d_);
        check(moe_synth_tokens(key, t0, n, d_, E, xh.data()));
        cuda_check(cudaMemcpy(R.x, xh.data(), sizeof(uint16_t) * n * d_, cudaMemcpyHostToDevice), "H2D x");
        cuda_check(cudaMemcpy(R.ids, ids.data() + t0 * k, sizeof(int32_t) * n * k, cudaMemcpyHostToDevice),
                   "H2D ids");
        check(moe_set_placement(R.layer->handle(), layer, rc.data(), rg.data()));
        st[r] = R.layer->forward_ids(layer, R.x, R.ids, nullptr, static_cast<int>(n), R.y, calls_);
      } catch (const std::exception& e) {
        err[r] = e.what();
      }
    };
    if (G_ == 1) {
      run_rank(0);
    } else {  // every rank enters the forward: the exchange handshakes need all of them
      std::vector<std::thread> th;
      for (int r = 0; r < G_; ++r) th.emplace_back(run_rank, r);
      for (auto& t : th) t.join();
    }
    for (int r = 0; r < G_; ++r)
      if (!err[r].empty()) throw std::runtime_error("rank " + std::to_string(r) + ": " + err[r]);
    // the straggler sets the layer time: max over ranks (cost_model.cpp:111-117)
    LayerMetrics m;
    double moe_ms = 0.0;
    for (const auto& s : st) {
      m.compute_ms = std::max(m.compute_ms, s.compute_ms);
      m.comm_ms = std::max(m.comm_ms, s.comm_ms);
      moe_ms = std::max(moe_ms, s.forward_ms);
    }
    // forward = measured MoE layer + the non-MoE part the reference charges
    // (t_misc: attention, norms), as in cost_model.cpp:114-121
    m.forward_ms = moe_ms + cluster.t_misc_ms;
    m.replica_count = plan.total_replicas();
    m.mem_mb = m.replica_count * model.expert_mem_mb;
    m.cost_mb_ms = moe_ms * m.mem_mb + cluster.t_misc_ms * cluster.m_misc_mb;
    last_ = st;
    return m;
  }

  const std::vector<moe_layer_stats>& last_stats() const { return last_; }

 private:
  struct Rank {
    std::unique_ptr<Layer> layer;
    uint16_t* x = nullptr;
    uint16_t* y = nullptr;
    int32_t* ids = nullptr;
    std::vector<char> loaded;  // per layer
  };

  static int env_int(const char* name, int def) {
    const char* v = std::getenv(name);
    return v && *v ? std::atoi(v) : def;
  }

  // contexts sized for `tokens` (re-created when a batch outgrows them) and
  // expert weights of `layer` loaded on every rank
  void ensure(int tokens, int layer) {
    const int per_rank = std::max(1, (tokens + G_ - 1) / G_);
    if (ranks_.empty() || per_rank > cap_) {
      release();
      cap_ = std::max(per_rank, 2 * cap_);
      ranks_.resize(G_);
      std::vector<moe_p2p_handle> handles(G_);
      for (int r = 0; r < G_; ++r) {
        cuda_check(cudaSetDevice(dev_[r]), "cudaSetDevice");
        ranks_[r].layer = std::make_unique<Layer>(model_, d_, ff_, cap_, G_, r, dev_[r]);
        cuda_check(cudaMalloc(&ranks_[r].x, sizeof(uint16_t) * cap_ * d_), "cudaMalloc");
        cuda_check(cudaMalloc(&ranks_[r].y, sizeof(uint16_t) * cap_ * d_), "cudaMalloc");
        cuda_check(cudaMalloc(&ranks_[r].ids, sizeof(int32_t) * cap_ * model_.top_k), "cudaMalloc");
        ranks_[r].loaded.assign(model_.num_layers, 0);
        if (G_ > 1) check(moe_p2p_export(ranks_[r].layer->handle(), &handles[r]));
      }
      if (G_ > 1)
        for (int r = 0; r < G_; ++r) check(moe_p2p_import(ranks_[r].layer->handle(), handles.data(), G_));
    }
    if (layer < 0 || layer >= model_.num_layers) throw std::invalid_argument("layer out of range");
    std::vector<uint16_t> w1, w3, w2;
    for (int r = 0; r < G_; ++r) {
      if (ranks_[r].loaded[layer]) continue;
      for (int e = 0; e < model_.experts_per_layer; ++e) {
        w1.resize(static_cast<size_t>(ff_) * d_);
        w3.resize(w1.size());
        w2.resize(w1.size());
        check(moe_synth_expert(moe_stream_key(seed_, layer, e, 0x65787074ull), d_, ff_, w1.data(), w3.data(),
                               w2.data()));
        ranks_[r].layer->load_expert(layer, e, w1.data(), w3.data(), w2.data());
      }
      ranks_[r].loaded[layer] = 1;
    }
  }

  void release() {
    for (auto& R : ranks_) {
      R.layer.reset();
      if (R.x) cudaFree(R.x);
      if (R.y) cudaFree(R.y);
      if (R.ids) cudaFree(R.ids);
    }
    ranks_.clear();
  }

 public:
  ~Engine() { release(); }

 private:
  ModelSpec model_;
  int d_ = 0, ff_ = 0, G_ = 1, cap_ = 0;
  uint64_t seed_ = 1;
  long calls_ = 0;
  std::vector<int> dev_;
  std::vector<Rank> ranks_;
  std::vector<moe_layer_stats> last_;
};

// Engine of the calling thread for a (cluster, model) — run_comparison runs
// run() on several threads at once (simulator.cpp:303-307), one context set
// each, as the C-ABI's one-context-per-thread rule asks.
inline Engine& engine(const ClusterSpec& cluster, const ModelSpec& model) {
  thread_local std::map<std::tuple<int, int, int, int>, std::unique_ptr<Engine>> engines;
  const auto key = std::make_tuple(cluster.gpu_count, model.num_layers, model.experts_per_layer, model.top_k);
  auto it = engines.find(key);
  if (it == engines.end()) it = engines.emplace(key, std::make_unique<Engine>(cluster, model)).first;
  return *it->second;
}

// The drop-in for LayerMetrics layer_forward_time(plan, placement, actual,
// cluster, model) (cost_model.hpp:24-26): the same arguments, the layer run
// for real on the B200(s).
inline LayerMetrics layer_forward_time(const ScalingPlan& plan, const Placement& placement, const LoadVector& actual,
                                       const ClusterSpec& cluster, const ModelSpec& model) {
  return engine(cluster, model).forward(plan, placement, actual, cluster, model);
}

}  // namespace moeless::b200
