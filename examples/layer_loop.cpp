// layer_loop.cpp — a reference-style C++ caller driving the B200 layer.
//
// Follows the per-layer body of the reference simulator's run()
// (proj/src/simulator.cpp:116-201) — predict -> scale_experts ->
// place_experts -> layer forward -> update_registry -> measure_accuracy — with
// the same moeless:: API, except that the analytic layer_forward_time is
// replaced by the real gate -> dispatch -> tcgen05 SwiGLU FFN -> combine on
// the GPU (moeless::b200::Layer, include/moeless/b200_layer.hpp).
//
//   layer_loop E k d_model d_ff tokens iterations
// prints one JSON line with p50/p99 (nearest rank, report.cpp:150-159) of the
// measured forward time and the predictor's realised accuracy.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "moe_b200.h"
#include "moeless/b200_layer.hpp"

using namespace moeless;

int main(int argc, char** argv) {
  const int E = argc > 1 ? std::atoi(argv[1]) : 8;
  const int k = argc > 2 ? std::atoi(argv[2]) : 2;
  const int d = argc > 3 ? std::atoi(argv[3]) : 1024;
  const int ff = argc > 4 ? std::atoi(argv[4]) : 3584;
  const int T = argc > 5 ? std::atoi(argv[5]) : 2048;
  const int iters = argc > 6 ? std::atoi(argv[6]) : 8;
  const std::uint64_t seed = 1;
  try {
    ModelSpec model;
    model.num_layers = 1;
    model.experts_per_layer = E;
    model.top_k = k;
    model.expert_mem_mb = 3.0 * d * ff * 2 / 1e6;
    model.layer_mem_cap_mb = 4 * model.expert_mem_mb;
    ClusterSpec cluster;
    cluster.gpu_count = 1;
    cluster.gpu_mem_capacity_mb = 180000.0;
    ScalerConfig scaler;
    PredictorProfile pp;
    pp.kind = PredictorKind::historical;  // plans from history, evaluated on actual
    pp.history_window = 8;

    b200::Layer layer(model, d, ff, T);
    std::vector<uint16_t> w1(static_cast<size_t>(d) * ff), w3(w1.size()), w2(w1.size());
    for (int e = 0; e < E; ++e) {
      b200::check(moe_synth_expert(moe_stream_key(seed, 0, e, 0x65787074), d, ff, w1.data(), w3.data(), w2.data()));
      layer.load_expert(0, e, w1.data(), w3.data(), w2.data());
    }
    const auto prof = make_popularity_profile(E, 1, 1.2, seed);
    const auto pop = popularity_weights(prof, 0, 0, Phase::prefill);
    std::vector<int32_t> noise(E);
    for (int e = 0; e < E; ++e) noise[e] = (e * 5 + 3) % E;
    std::vector<uint16_t> wg(static_cast<size_t>(E) * d);
    b200::check(moe_synth_gate(moe_stream_key(seed, 0, 0, 0x67617465), d, E, pop.data(), noise.data(), wg.data()));
    layer.set_gate(0, wg.data());

    std::vector<uint16_t> xh(static_cast<size_t>(T) * d);
    uint16_t *x = nullptr, *y = nullptr;
    if (cudaMalloc(&x, xh.size() * 2) != cudaSuccess || cudaMalloc(&y, xh.size() * 2) != cudaSuccess)
      throw std::runtime_error("cudaMalloc failed");

    ReplicaRegistry registry(50);
    std::vector<LoadVector> history;
    std::vector<double> forwards;
    double acc_sum = 0.0;
    for (long it = 0; it < iters; ++it) {
      b200::check(moe_synth_tokens(moe_stream_key(seed, it, 0, 0x78746f6b), 0, T, d, E, xh.data()));
      cudaMemcpy(x, xh.data(), xh.size() * 2, cudaMemcpyHostToDevice);
      LoadVector known{0, std::vector<std::int64_t>(E, 0)};
      known.loads[0] = static_cast<std::int64_t>(T) * k;  // the historical predictor reads only the total
      const LoadVector predicted = predict(known, history, pp, it, seed);
      const ScalingPlan plan = scale_experts(predicted, model, scaler);
      const PlaceResult placed = place_experts(plan, cluster, registry, it);
      const b200::ForwardResult r = layer.forward(plan, placed.placement, x, T, y, it);
      update_registry(registry, placed.placement, it);
      acc_sum += measure_accuracy(predicted, r.actual);
      history.push_back(r.actual);
      forwards.push_back(r.metrics.forward_ms);
    }
    std::printf(
        "{\"E\": %d, \"k\": %d, \"d\": %d, \"ff\": %d, \"tokens\": %d, \"iterations\": %d, \"p50_ms\": %.4f, "
        "\"p99_ms\": %.4f, \"mean_accuracy\": %.4f, \"tokens_per_s_p50\": %.1f}\n",
        E, k, d, ff, T, iters, percentile(forwards, 0.5), percentile(forwards, 0.99), acc_sum / iters,
        T / (percentile(forwards, 0.5) * 1e-3));
    cudaFree(x);
    cudaFree(y);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "layer_loop: %s\n", e.what());
    return 1;
  }
  return 0;
}
