// moeless/b200_layer.hpp — header-only C++ shim over the C-ABI (moe_b200.h).
//
// This is the binding a maintainer of the reference adds to reach the GPU
// from its C++ API: value types in, value types out, status codes turned back
// into the exceptions the reference throws (std::invalid_argument for bad
// input, std::runtime_error for infeasible placement / CUDA / NCCL), and the
// reference's call sequence kept intact:
//
//   auto plan      = moeless::scale_experts(predicted, model, scaler);      // scaler.hpp:29
//   auto placed    = moeless::place_experts(plan, cluster, registry, it);   // placer.hpp:74
//   LayerMetrics m = layer.forward(plan, placed.placement, x, T, y, it);    // replaces
//                    // layer_forward_time(plan, placement, actual, cluster, model) (cost_model.hpp:24)
//   moeless::update_registry(registry, placed.placement, it);                // placer.hpp:80
//
// `actual` is no longer an input: the layer's gate produces it (route_tokens'
// role, workload.hpp:90) and it is returned in LayerMetrics-compatible stats.
#pragma once

#include <stdexcept>
#include <string>
#include <vector>

#include "moe_b200.h"
#include "moeless/api.hpp"

namespace moeless::b200 {

inline void check(int rc) {
  if (rc == MOE_OK) return;
  const std::string msg = moe_last_error();
  if (rc == MOE_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

struct ForwardResult {
  LayerMetrics metrics;       // measured compute / comm / forward ms, replicas, memory
  moe_layer_stats stats;      // per-phase device times and this rank's gate histogram
  LoadVector actual;          // the gate's per-expert loads (what route_tokens modelled)
};

class Layer {
 public:
  // One rank of an MoE layer stack on one B200.  `model.num_layers`,
  // `experts_per_layer`, `top_k` come from the reference ModelSpec.
  Layer(const ModelSpec& model, int d_model, int d_ff, int max_tokens, int world_size = 1, int rank = 0,
        int device = 0, const void* nccl_unique_id = nullptr) {
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
    d.exchange_mode = MOE_EXCHANGE_NCCL;
    d.nccl_unique_id = nccl_unique_id;
    d.expert_mem_mb = model.expert_mem_mb;
    d.layer_mem_cap_mb = model.layer_mem_cap_mb;
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

  // Flattens ScalingPlan.replica_counts (types.hpp:59) and Placement.gpu_for
  // (placer.hpp:17) into the C-ABI replica table.
  void set_placement(const ScalingPlan& plan, const Placement& placement) {
    std::vector<int32_t> rc(plan.replica_counts.begin(), plan.replica_counts.end());
    std::vector<int32_t> rg;
    for (const auto& per : placement.gpu_for) rg.insert(rg.end(), per.begin(), per.end());
    check(moe_set_placement(ctx_, plan.layer, rc.data(), rg.data()));
  }

  // The real layer forward for a (plan, placement) pair: device buffers in/out.
  ForwardResult forward(const ScalingPlan& plan, const Placement& placement, const uint16_t* x_dev, int tokens,
                        uint16_t* y_dev, long iteration, void* stream = nullptr) {
    set_placement(plan, placement);
    ForwardResult r{};
    check(moe_layer_forward(ctx_, plan.layer, x_dev, tokens, y_dev, MOE_PLAN_FIXED, iteration, &r.stats, stream));
    fill(r, plan.layer);
    return r;
  }

  // Same, with the MoEless planner run on the layer's own gate histogram
  // (oracle predictor, distance 0) inside the call.
  ForwardResult forward_planned(int layer, const uint16_t* x_dev, int tokens, uint16_t* y_dev, long iteration,
                                void* stream = nullptr) {
    ForwardResult r{};
    check(moe_layer_forward(ctx_, layer, x_dev, tokens, y_dev, MOE_PLAN_SYNC, iteration, &r.stats, stream));
    fill(r, layer);
    return r;
  }

  moe_ctx* handle() const { return ctx_; }

 private:
  void fill(ForwardResult& r, int layer) const {
    r.metrics.compute_ms = r.stats.compute_ms;
    r.metrics.comm_ms = r.stats.comm_ms;
    r.metrics.forward_ms = r.stats.forward_ms;
    r.metrics.replica_count = r.stats.replica_count;
    r.metrics.mem_mb = r.stats.mem_mb;
    r.metrics.cost_mb_ms = (r.stats.compute_ms + 2.0 * r.stats.comm_ms) * r.stats.mem_mb;
    r.actual.layer = layer;
    r.actual.loads.assign(r.stats.counts, r.stats.counts + E_);
  }
  moe_ctx* ctx_ = nullptr;
  int E_ = 0;
};

}  // namespace moeless::b200
