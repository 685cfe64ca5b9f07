// gate_common.cuh — device helpers shared by the gate (gate.cu) and the fused
// decode front end (frontend.cu): the m16n8k16 fragment MMA, the warp arg-max
// top-k with lower-index tie-breaking, and the predictor-MLP scoring.
#pragma once
#include <cfloat>
#include <cstdint>

#include "sm100_ptx.cuh"

namespace moe {
namespace {

constexpr int kBlockTokens = 32;  // tokens per CTA == per block_counts row
constexpr int kWarps = 8;
constexpr int kSlices = 4;        // K-slices per m-tile inside a CTA
constexpr int kPerLane = 8;       // stacked logits per lane in the top-k (<= 256)
constexpr int kMaxHistExperts = 256;
#ifndef MOE_GATE_UNROLL
#define MOE_GATE_UNROLL 2
#endif
constexpr int kGateUnroll = MOE_GATE_UNROLL;  // K-loop iterations in flight per warp (two 16-byte x loads each)

__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                               uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// Top-k over logits [base, base+E) of one token's stacked row in shared
// memory; lane l looks at l, l+32, ...  Every lane returns the same result.
// Top-k over per-lane values own[s] = value of expert lane + 32 s.
// S = logits per lane actually held (ceil(columns / 32)): the decode shape
// (64 experts) scans 2 slots per round, not kPerLane.
// Order-preserving 32-bit key of a logit (larger float <-> larger key, -0 ==
// +0); NaN maps to 1, below every number, and 0 marks a slot out of the race.
__device__ __forceinline__ uint32_t logit_key(float f) {
  if (f != f) return 1u;
  uint32_t u = __float_as_uint(f);
  if ((u << 1) == 0u) u = 0u;
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key_logit(uint32_t key) {
  return __uint_as_float((key & 0x80000000u) ? (key & 0x7fffffffu) : ~key);
}

// Per round, the warp's largest key is one redux.sync max and the lowest expert
// holding it one redux.sync min (ties -> lower index, as the arg-max with
// `v > best || (v == best && e < bi)` it replaces), instead of a 5-step
// value + index shuffle butterfly: the k rounds are a chain of 2 reductions.
template <int S>
__device__ __forceinline__ void warp_topk_vals(const float (&own)[S], int E, int k, int (&ids_out)[8],
                                               float (&logit_out)[8]) {
  const int lane = lane_id();
  uint32_t key[S];
#pragma unroll
  for (int s = 0; s < S; ++s) key[s] = lane + 32 * s < E ? logit_key(own[s]) : 0u;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    if (j >= k) break;
    uint32_t best = 0u, be = 0xffffffffu;
#pragma unroll
    for (int s = 0; s < S; ++s)
      if (key[s] > best) { best = key[s]; be = lane + 32 * s; }  // first s: the lane's lowest expert
    const uint32_t kmax = __reduce_max_sync(0xffffffffu, best);
    const uint32_t emin = __reduce_min_sync(0xffffffffu, best == kmax ? be : 0xffffffffu);
#pragma unroll
    for (int s = 0; s < S; ++s)
      if (emin == static_cast<uint32_t>(lane + 32 * s)) key[s] = 0u;
    ids_out[j] = static_cast<int>(emin);
    logit_out[j] = key_logit(kmax);
  }
}

template <int S>
__device__ __forceinline__ void warp_topk(const float* row, int base, int E, int k, int (&ids_out)[8],
                                          float (&logit_out)[8]) {
  const int lane = lane_id();
  float own[S];
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int e = lane + 32 * s;
    own[s] = e < E ? row[base + e] : -FLT_MAX;
  }
  warp_topk_vals(own, E, k, ids_out, logit_out);
}

// The batched predictor MLP (K2 with a hidden layer): its E hidden units are
// the slot's stacked rows (computed in the same read of x as the gate), so
// per token the warp turns them in place into out[e] = sum_j W2[e][j]
// relu(hidden_j) — an fmaf chain in j order, reproducible bit for bit on the
// CPU — and the usual top-k runs on out.  W2 [E][E] fp32 per slot.  A
// separate instantiation (MLP = true): the linear path keeps its registers.
struct PredictorMlp {
  const float* w2;  // [n_pred][E][E]; nullptr: every slot linear
  uint32_t mask;    // bit p: slot p is an MLP
};

template <int S>
__device__ __forceinline__ void mlp_scores_inplace(float* seg, int E, const float* __restrict__ w2) {
  const int lane = lane_id();
  float own[S];
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int e = lane + 32 * s;
    float acc = 0.0f;
    if (e < E) {
      const float* w = w2 + (size_t)e * E;
      for (int j = 0; j < E; ++j) {
        const float h = seg[j];
        acc = fmaf(__ldg(w + j), h > 0.0f ? h : 0.0f, acc);
      }
    }
    own[s] = acc;
  }
  __syncwarp();
#pragma unroll
  for (int s = 0; s < S; ++s)
    if (lane + 32 * s < E) seg[lane + 32 * s] = own[s];
  __syncwarp();
}


// Split-K partial logits of one 32-token block: the CTA (8 warps) covers the
// K range [split * d / nsplit, (split + 1) * d / nsplit); warp w takes m-tile
// (w & 1) (16 tokens) and K-slice (w >> 1) of it, so a CTA keeps 8
// independent 16-byte-load streams in flight.  Fragments come straight from
// global memory: the 16 k-slots of one MMA are mapped to features so that
// lane (g, c) needs 4 CONSECUTIVE features of row g / row g+8 / expert g
// (slots 2c,2c+1 <-> f, f+1 and 2c+8,2c+9 <-> f+2, f+3, identical for A and
// B), i.e. one 16-byte load per row feeds two MMAs.  The 4 K-slices are summed
// into red[32][8 NT + 4] in a fixed order (deterministic); ends with the CTA
// synchronised.  d / (kSlices * nsplit) must be a multiple of 32.
template <int NT>
__device__ __forceinline__ void block_partial_logits(const __nv_bfloat16* __restrict__ x, int T, int d,
                                                     const __nv_bfloat16* __restrict__ w_all, int Etot, int blk,
                                                     int split, int nsplit, float* red) {
  constexpr int kLd = 8 * NT + 4;
  const int warp = threadIdx.x >> 5, lane = lane_id();
  const int g = lane >> 2, c = lane & 3;
  const int mt = warp & 1, ks = warp >> 1;
  // ---- skinny GEMM: 16 tokens x 8*NT logits over this warp's K-slice
  const int r0 = blk * kBlockTokens + mt * 16 + g, r1 = r0 + 8;
  const bool v0 = r0 < T, v1 = r1 < T;
  const __nv_bfloat16* x0 = x + (size_t)(v0 ? r0 : 0) * d;
  const __nv_bfloat16* x1 = x + (size_t)(v1 ? r1 : 0) * d;
  const int slice = d / (kSlices * nsplit);  // multiple of 32 (checked by the launcher)
  const int k_begin = (split * kSlices + ks) * slice, k_end = k_begin + slice;
  float acc[NT][4];
#pragma unroll
  for (int n = 0; n < NT; ++n) acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.0f;
  const int4 zero = make_int4(0, 0, 0, 0);
#pragma unroll kGateUnroll
  for (int kb = k_begin; kb < k_end; kb += 32) {
    const int f = kb + 8 * c;  // this lane's 8 consecutive features of the 32-feature block
    const int4 a_lo = v0 ? ld_nc_v4(x0 + f) : zero;
    const int4 a_hi = v1 ? ld_nc_v4(x1 + f) : zero;
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      const int e = n * 8 + g;
      const int4 b = e < Etot ? __ldg(reinterpret_cast<const int4*>(w_all + (size_t)e * d + f)) : zero;
      mma_bf16_16816(acc[n], a_lo.x, a_hi.x, a_lo.y, a_hi.y, b.x, b.y);  // features f .. f+3
      mma_bf16_16816(acc[n], a_lo.z, a_hi.z, a_lo.w, a_hi.w, b.z, b.w);  // features f+4 .. f+7
    }
  }
  // ---- ordered K-slice reduction into shared memory (deterministic)
  for (int s = 0; s < kSlices; ++s) {
    if (ks == s) {
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        float* p0 = red + (mt * 16 + g) * kLd + n * 8 + 2 * c;
        float* p1 = p0 + 8 * kLd;
        if (s == 0) {
          p0[0] = acc[n][0]; p0[1] = acc[n][1]; p1[0] = acc[n][2]; p1[1] = acc[n][3];
        } else {
          p0[0] += acc[n][0]; p0[1] += acc[n][1]; p1[0] += acc[n][2]; p1[1] += acc[n][3];
        }
      }
    }
    __syncthreads();
  }
}

}  // namespace
}  // namespace moe
