// synth.cpp — deterministic synthetic layer inputs for the bench and tests
// (DESIGN.md §"Synthetic inputs").  No dataset or checkpoint exists offline,
// so inputs are generated from counter-based streams keyed like the
// reference's keyed_engine (rng.hpp:21-25) and placed on a grid where every
// fp32 gate logit is exact in any summation order:
//   x   : col 0 = 1 (bias feature); cols 1..E = Gumbel noise on a 1/16 grid
//         (|q| <= 255, exact in bf16); other cols q/16, |q| <= 16.
//   Wg  : col 0 = round(16 ln w_e)/16 (Zipf log-popularity, workload.cpp:77-88);
//         col 1+noise_perm[e] = 1; other cols q/4096, |q| <= 16.
// Products are multiples of 2^-16 and every partial sum stays below 2^6, so
// the 24-bit fp32 significand holds them exactly: ids and counts are
// bit-identical between the GPU kernel and the CPU oracle, and Gumbel-top-k
// of ln w + G draws k distinct experts with route_tokens' distribution.
#include <cmath>
#include <cstdint>
#include <cstring>

#include "host/moeless_api.hpp"

namespace moe {

namespace {
constexpr uint64_t kStep = 0xD1B54A32D192ED03ULL;

inline uint64_t stream_value(uint64_t key, uint64_t i) { return moeless::mix64(key ^ (i * kStep)); }

inline uint16_t to_bf16(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) return static_cast<uint16_t>((u >> 16) | ((u & 0xffffu) ? 0x40u : 0u));
  u += 0x7fffu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

// Gumbel(0,1) quantised to 1/16, clamped to |q| <= 255.
inline int gumbel16(uint64_t r) {
  const double u = (static_cast<double>(r >> 11) + 0.5) * 0x1.0p-53;
  long q = std::lrint(-std::log(-std::log(u)) * 16.0);
  return static_cast<int>(q > 255 ? 255 : (q < -255 ? -255 : q));
}
}  // namespace

uint64_t stream_key(uint64_t seed, uint64_t a, uint64_t b, uint64_t tag) {
  return moeless::mix64(seed ^ moeless::mix64(a ^ moeless::mix64(b ^ moeless::mix64(tag))));
}

void synth_tokens(uint64_t key, int64_t first, int64_t tokens, int d, int E, uint16_t* x) {
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < tokens; ++t) {
    const int64_t gt = first + t;
    uint16_t* row = x + t * d;
    row[0] = to_bf16(1.0f);
    for (int c = 1; c < d; ++c) {
      const uint64_t r = stream_value(key, static_cast<uint64_t>(gt * d + c));
      const float v = c <= E ? static_cast<float>(gumbel16(r)) / 16.0f
                             : static_cast<float>(static_cast<int>(r % 33) - 16) / 16.0f;
      row[c] = to_bf16(v);
    }
  }
}

void synth_gate(uint64_t key, int d, int E, const double* pop, const int32_t* noise_perm, uint16_t* wg) {
  for (int e = 0; e < E; ++e) {
    uint16_t* row = wg + static_cast<int64_t>(e) * d;
    long q = std::lrint(std::log(pop[e]) * 16.0);
    row[0] = to_bf16(static_cast<float>(q < -255 ? -255 : q) / 16.0f);
    for (int c = 1; c < d; ++c) {
      float v;
      if (c <= E) {
        v = (c - 1 == noise_perm[e]) ? 1.0f : 0.0f;
      } else {
        const uint64_t r = stream_value(key, static_cast<uint64_t>(static_cast<int64_t>(e) * d + c));
        v = static_cast<float>(static_cast<int>(r % 33) - 16) / 4096.0f;
      }
      row[c] = to_bf16(v);
    }
  }
}

void synth_expert(uint64_t key, int d, int ff, uint16_t* w1, uint16_t* w3, uint16_t* w2) {
  const float s1 = 1.0f / std::sqrt(static_cast<float>(d));
  const float s2 = 1.0f / std::sqrt(static_cast<float>(ff));
  const int64_t n = static_cast<int64_t>(d) * ff;
  auto q64 = [&](uint64_t i) { return static_cast<float>(static_cast<int>(stream_value(key, i) % 129) - 64) / 64.0f; };
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    w1[i] = to_bf16(q64(static_cast<uint64_t>(i)) * s1);
    w3[i] = to_bf16(q64(static_cast<uint64_t>(n + i)) * s1);
    w2[i] = to_bf16(q64(static_cast<uint64_t>(2 * n + i)) * s2);
  }
}

}  // namespace moe
