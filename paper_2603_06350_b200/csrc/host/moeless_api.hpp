// host/moeless_api.hpp — INTERNAL declarations of the library's host planner:
// a restatement, inside libmoe_b200.so, of the reference's planning functions
// (/root/reference/proj/include/moeless/*.hpp: scale_experts, place_experts,
// ReplicaRegistry, predict, layer_forward_time, route_tokens, static_plan, ...)
// that the context runs for MOE_PLAN_SYNC / MOE_PLAN_PREDICTED and that the
// C-ABI exports as moe_plan_* entry points.  Implementation: planner.cpp.
//
// This header is NOT installed and does not replace the reference's headers:
// reference callers keep compiling against proj/include/moeless and reach the
// GPU through include/moeless/b200_layer.hpp (C-ABI only).  The library
// exports only the moe_* C symbols (csrc/exports.map), so these C++ symbols
// never clash with a reference build linked into the same program.
//
// Behavioural contract kept from the reference:
//   * bad arguments throw std::invalid_argument, infeasible placements throw
//     std::runtime_error naming the replica ("no GPU has memory for replica
//     (e,r) of layer l", placer.cpp:100-104);
//   * every decision that the reference takes on exact rationals or on a
//     specific floating-point expression is reproduced with the same
//     arithmetic, so plans are bit-identical (tests/test_planner_parity.py).
#pragma once

#include <cstdint>
#include <map>
#include <numeric>
#include <optional>
#include <random>
#include <stdexcept>
#include <string>
#include <tuple>
#include <utility>
#include <vector>

namespace moeless {

// ------------------------------------------------------------ rational.hpp
// Exact non-negative-denominator fraction; ordering by 128-bit cross products
// (reference: rational.hpp:15-55).  Shares w/r stay exact so heap order and
// sort order never depend on rounding.
struct Rational {
  std::int64_t num = 0;
  std::int64_t den = 1;

  constexpr Rational() = default;
  Rational(std::int64_t n, std::int64_t d = 1) : num(n), den(d) { reduce(); }

  void reduce() {
    if (den == 0) throw std::invalid_argument("rational with zero denominator");
    if (den < 0) { num = -num; den = -den; }
    std::int64_t g = std::gcd(num < 0 ? -num : num, den);
    if (g > 1) { num /= g; den /= g; }
  }
  void normalize() { reduce(); }
  double to_double() const { return static_cast<double>(num) / static_cast<double>(den); }

  Rational operator+(const Rational& o) const { return {num * o.den + o.num * den, den * o.den}; }
  Rational operator-(const Rational& o) const { return {num * o.den - o.num * den, den * o.den}; }
  bool operator==(const Rational& o) const { return num == o.num && den == o.den; }
  bool operator!=(const Rational& o) const { return !(*this == o); }
  bool operator<(const Rational& o) const {
    return static_cast<__int128>(num) * o.den < static_cast<__int128>(o.num) * den;
  }
  bool operator>(const Rational& o) const { return o < *this; }
  bool operator<=(const Rational& o) const { return !(o < *this); }
  bool operator>=(const Rational& o) const { return !(*this < o); }
};

// ----------------------------------------------------------------- rng.hpp
// splitmix64 finaliser and keyed mt19937_64 streams (rng.hpp:12-32).
std::uint64_t mix64(std::uint64_t x);
std::mt19937_64 keyed_engine(std::uint64_t seed, std::uint64_t a, std::uint64_t b,
                             std::uint64_t tag);
inline double uniform01(std::mt19937_64& eng) { return (eng() >> 11) * 0x1.0p-53; }

// --------------------------------------------------------------- types.hpp
struct ClusterSpec {
  int gpu_count = 1;
  double gpu_mem_capacity_mb = 48000.0;
  double alpha_ms_per_token = 0.01;
  double beta_ms_per_token = 0.002;
  double t_misc_ms = 0.5;
  double m_misc_mb = 0.0;
  void validate() const;
};

struct ModelSpec {
  int num_layers = 2;
  int experts_per_layer = 1;
  int top_k = 1;
  double expert_mem_mb = 330.0;
  double layer_mem_cap_mb = 0.0;
  void validate() const;
};

struct LoadVector {
  int layer = 0;
  std::vector<std::int64_t> loads;
  std::int64_t total() const { return std::accumulate(loads.begin(), loads.end(), std::int64_t{0}); }
};

struct ReplicaShare {
  int expert = 0;
  int ordinal = 0;
  Rational share;
};

struct ScalingPlan {
  int layer = 0;
  std::vector<int> replica_counts;
  std::vector<ReplicaShare> shares;  // (expert, ordinal) order
  double alloc_mem_mb = 0.0;
  double expert_mem_mb = 0.0;
  int total_replicas() const { return std::accumulate(replica_counts.begin(), replica_counts.end(), 0); }
};

struct LayerMetrics {
  double compute_ms = 0.0;
  double comm_ms = 0.0;
  double forward_ms = 0.0;
  int replica_count = 0;
  double mem_mb = 0.0;
  double cost_mb_ms = 0.0;
};

// ------------------------------------------------------------ workload.hpp
enum class Phase { prefill, decode };

struct IterationBatch {
  long iteration = 0;
  Phase phase = Phase::prefill;
  std::int64_t token_count = 0;
};

struct PopularityProfile {
  std::vector<std::vector<int>> rank_to_expert;
  double zipf_exponent = 1.2;
  double zipf_exponent_decode = -1.0;
  int drift_period = 0;
  std::uint64_t perm_seed = 0;
  int num_layers() const { return static_cast<int>(rank_to_expert.size()); }
  int num_experts() const { return rank_to_expert.empty() ? 0 : static_cast<int>(rank_to_expert[0].size()); }
  double exponent_for(Phase p) const {
    return (p == Phase::decode && zipf_exponent_decode >= 0.0) ? zipf_exponent_decode : zipf_exponent;
  }
};

PopularityProfile make_popularity_profile(int experts, int layers, double zipf_exponent,
                                          std::uint64_t seed, bool shared_permutation = false,
                                          int drift_period = 0, double zipf_exponent_decode = -1.0);
std::vector<int> effective_permutation(const PopularityProfile& profile, int layer, long iteration);
std::vector<double> popularity_weights(const PopularityProfile& profile, int layer, long iteration,
                                       Phase phase);
LoadVector route_tokens(const IterationBatch& batch, int layer, const PopularityProfile& profile,
                        int top_k, int experts, std::uint64_t seed);

// ----------------------------------------------------------- predictor.hpp
enum class PredictorKind { oracle, noisy, historical };

struct PredictorProfile {
  PredictorKind kind = PredictorKind::noisy;
  int distance = 1;
  std::vector<double> per_layer_accuracy;
  double accuracy_threshold = 0.8;
  double distance_decay = 0.04;
  int history_window = 8;
  std::vector<bool> fine_tuned;
  double effective_accuracy(int layer) const;
  void validate(int num_layers) const;
};

PredictorProfile make_ramp_profile(int num_layers, double first, double last);
LoadVector predict(const LoadVector& actual_future, const std::vector<LoadVector>& history,
                   const PredictorProfile& profile, long iteration, std::uint64_t seed,
                   const std::vector<double>& popularity = {}, bool* bootstrap_fallback = nullptr);
double measure_accuracy(const LoadVector& predicted, const LoadVector& actual);
void apply_layer_aware_finetuning(PredictorProfile& profile);

// -------------------------------------------------------------- scaler.hpp
struct ScalerConfig {
  double cv_threshold = 0.2;
  bool exclude_zero_loads_from_cv = false;
};

struct ScaleTrace {
  std::vector<int> split_expert;
  std::vector<Rational> max_share;
  std::vector<double> cv;
};

ScalingPlan scale_experts(const LoadVector& predicted, const ModelSpec& model,
                          const ScalerConfig& config, ScaleTrace* trace = nullptr);

struct VerifyReport {
  bool ok = true;
  std::vector<std::string> issues;
};
VerifyReport verify_plan(const ScalingPlan& plan, const LoadVector& predicted,
                         const ModelSpec& model, const ScalerConfig& config);

// -------------------------------------------------------------- placer.hpp
struct Placement {
  int layer = 0;
  std::vector<std::vector<int>> gpu_for;  // [expert][ordinal] -> gpu
  std::vector<double> per_gpu_mem_mb;
  int gpu_count() const { return static_cast<int>(per_gpu_mem_mb.size()); }
};

struct PlaceResult {
  Placement placement;
  int warm_count = 0;
  int cold_count = 0;
};

struct PlacerOptions {
  bool load_includes_compute = false;
  double alpha_ms_per_token = 0.0;
  double beta_ms_per_token = 1.0;
};

class ReplicaRegistry {
 public:
  struct Entry {
    int gpu = 0;
    long last_used = 0;
  };
  explicit ReplicaRegistry(int keep_alive_iters = 0);
  int keep_alive_iters() const { return keep_alive_; }
  std::optional<int> lookup(int layer, int expert, int ordinal, long iteration) const;
  void record(int layer, int expert, int ordinal, int gpu, long iteration);
  void retire(int layer, const Placement& placement, long iteration);
  std::size_t size() const { return live_.size(); }

 private:
  int keep_alive_;
  std::map<std::tuple<int, int, int>, Entry> live_;
};

PlaceResult place_experts(const ScalingPlan& plan, const ClusterSpec& cluster,
                          const ReplicaRegistry& registry, long iteration,
                          const PlacerOptions& options = {});
void update_registry(ReplicaRegistry& registry, const Placement& placement, long iteration);

// ---------------------------------------------------------- cost_model.hpp
double replica_time(double load_share_tokens, double alpha_ms_per_token);
std::vector<double> gpu_comm_times(const ScalingPlan& plan, const Placement& placement,
                                   double beta_ms_per_token);
LayerMetrics layer_forward_time(const ScalingPlan& plan, const Placement& placement,
                                const LoadVector& actual, const ClusterSpec& cluster,
                                const ModelSpec& model);
double coefficient_of_variation(const std::vector<double>& values);
double serverful_cost(double total_ms, const ModelSpec& model, const ClusterSpec& cluster);

// ----------------------------------------------------------- baselines.hpp
std::pair<ScalingPlan, Placement> static_plan(const LoadVector& loads, const ModelSpec& model,
                                              const ClusterSpec& cluster);
LayerMetrics oracle_balance_time(const LoadVector& actual, const ClusterSpec& cluster,
                                 const ModelSpec& model);
// replica f (flattened (expert, ordinal)) -> GPU f mod G: the simulator's
// static_rr placement ablation (simulator.cpp:32-50)
Placement round_robin_placement(const ScalingPlan& plan, const ClusterSpec& cluster);

// -------------------------------------------------------------- report.hpp
double percentile(std::vector<double> values, double q);

}  // namespace moeless
