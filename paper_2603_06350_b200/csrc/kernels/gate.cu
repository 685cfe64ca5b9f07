// gate.cu — K1: fused gate GEMV + softmax + top-k + per-expert histogram,
// with the K2 load predictor fused into the same read of x.
//
// Replaces the routing stand-in route_tokens (reference
// proj/src/workload.cpp:188-230): instead of sampling, every token's experts
// come from its own activations.  Conventions: logits = x Wg^T
// accumulated in fp32; the k largest logits are taken by repeated arg-max with
// the LOWER expert index winning ties; weights are the softmax over E
// restricted to the chosen k (== softmax over the k logits); counts[e] is the
// histogram of chosen experts (sum == T*k, as route_tokens guarantees).
//
// Work decomposition: one warp owns a block of 32 consecutive tokens (this is
// also the granularity of block_counts[], the stable prefix the dispatch
// kernel scans).  Each lane owns 8 contiguous columns per 256-column step, so
// x is read with one 16-byte L1-bypassing load per lane per step (512 B
// coalesced per warp) and each weight vector is reused for TOKG tokens.
// Partial sums are all-reduced with xor shuffles; lane (e mod 32) keeps
// expert e for the arg-max and for the histogram, which is flushed with one
// global atomicAdd per (block, expert).
//
// The predictor weights (n_pred target layers, each [E, d]) are stacked under
// the gate weights: the same pass over x yields pred_counts[p][E] (histogram
// only), so K2 costs no extra HBM read of x while E*(1+n_pred) <= EC.
#include <cfloat>
#include <cstdint>

#include "sm100_ptx.cuh"

namespace moe {

namespace {

constexpr int kWarpsPerCta = 4;
constexpr int kBlockTokens = 32;  // tokens per warp == per block_counts row
constexpr int kPerLane = 8;       // stacked experts per lane -> E*(1+n_pred) <= 256

// Top-k over the experts [base, base+E) of a stacked logit vector held as
// lane l -> stacked index l + 32 s.  Every lane returns the same ids/logits.
__device__ __forceinline__ void warp_topk(const float (&own)[kPerLane], int base, int E, int k,
                                          int* ids_out, float* logit_out) {
  const int lane = lane_id();
  uint32_t taken = 0;
  for (int j = 0; j < k; ++j) {
    float bv = -FLT_MAX;
    int bi = 0x7fffffff;
#pragma unroll
    for (int s = 0; s < kPerLane; ++s) {
      const int e = lane + 32 * s - base;
      if (e >= 0 && e < E && !((taken >> s) & 1u))
        if (own[s] > bv || (own[s] == bv && e < bi)) { bv = own[s]; bi = e; }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    const int st = bi + base;
    if ((st & 31) == lane) taken |= 1u << (st >> 5);
    ids_out[j] = bi;
    logit_out[j] = bv;
  }
}

}  // namespace

// x [T, d] bf16; w_all [(1 + n_pred) * E, d] bf16 (rows 0..E-1 = gate).
// Outputs: ids [T, k] i32, weights [T, k] f32, counts [E] i32 (atomic; caller
// zeroes), block_counts [ceil(T/32), E] i32, pred_counts [n_pred, E] (atomic).
template <int TOKG, int EC>
__global__ void __launch_bounds__(kWarpsPerCta * 32)
gate_topk_kernel(const __nv_bfloat16* __restrict__ x, int T, int d,
                 const __nv_bfloat16* __restrict__ w_all, int E, int n_pred, int k,
                 int32_t* __restrict__ ids, float* __restrict__ wts, int32_t* __restrict__ counts,
                 int32_t* __restrict__ block_counts, int32_t* __restrict__ pred_counts) {
  const int warp = threadIdx.x >> 5;
  const int lane = lane_id();
  const int blk = blockIdx.x * kWarpsPerCta + warp;
  const int t_begin = blk * kBlockTokens;
  if (t_begin >= T) return;
  const int t_end = min(T, t_begin + kBlockTokens);
  const int Etot = E * (1 + n_pred);

  int hist[kPerLane];  // gate histogram for stacked index lane + 32 s (< E)
#pragma unroll
  for (int s = 0; s < kPerLane; ++s) hist[s] = 0;

  for (int t0 = t_begin; t0 < t_end; t0 += TOKG) {
    const int ntok = min(TOKG, t_end - t0);
    float own[TOKG][kPerLane];
#pragma unroll
    for (int q = 0; q < TOKG; ++q)
#pragma unroll
      for (int s = 0; s < kPerLane; ++s) own[q][s] = -FLT_MAX;

    for (int e0 = 0; e0 < Etot; e0 += EC) {
      float acc[TOKG][EC];
#pragma unroll
      for (int q = 0; q < TOKG; ++q)
#pragma unroll
        for (int c = 0; c < EC; ++c) acc[q][c] = 0.0f;

      for (int col = lane * 8; col < d; col += 256) {
        float xv[TOKG][8];
#pragma unroll
        for (int q = 0; q < TOKG; ++q) {
          int4 raw = make_int4(0, 0, 0, 0);
          if (q < ntok) raw = ld_nc_v4(x + (size_t)(t0 + q) * d + col);
          const uint32_t* u = reinterpret_cast<const uint32_t*>(&raw);
#pragma unroll
          for (int i = 0; i < 4; ++i) { xv[q][2 * i] = bf16lo(u[i]); xv[q][2 * i + 1] = bf16hi(u[i]); }
        }
#pragma unroll
        for (int c = 0; c < EC; ++c) {
          if (e0 + c < Etot) {
            const int4 raw = __ldg(reinterpret_cast<const int4*>(w_all + (size_t)(e0 + c) * d + col));
            const uint32_t* u = reinterpret_cast<const uint32_t*>(&raw);
            float wv[8];
#pragma unroll
            for (int i = 0; i < 4; ++i) { wv[2 * i] = bf16lo(u[i]); wv[2 * i + 1] = bf16hi(u[i]); }
#pragma unroll
            for (int q = 0; q < TOKG; ++q)
#pragma unroll
              for (int i = 0; i < 8; ++i) acc[q][c] = fmaf(xv[q][i], wv[i], acc[q][c]);
          }
        }
      }
#pragma unroll
      for (int q = 0; q < TOKG; ++q)
#pragma unroll
        for (int c = 0; c < EC; ++c) {
          float v = acc[q][c];
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
          const int st = e0 + c;
          if (st < Etot && (st & 31) == lane) {
#pragma unroll
            for (int s = 0; s < kPerLane; ++s)
              if ((st >> 5) == s) own[q][s] = v;
          }
        }
    }

#pragma unroll
    for (int q = 0; q < TOKG; ++q) {
      if (q < ntok) {
        const int t = t0 + q;
        for (int g = 0; g <= n_pred; ++g) {
          int sel[8];
          float lg[8];
          warp_topk(own[q], g * E, E, k, sel, lg);
          if (g == 0) {
            if (lane == 0) {
              float z = 0.0f, p[8];
              for (int j = 0; j < k; ++j) { p[j] = expf(lg[j] - lg[0]); z += p[j]; }
              for (int j = 0; j < k; ++j) {
                ids[(size_t)t * k + j] = sel[j];
                wts[(size_t)t * k + j] = p[j] / z;
              }
            }
            for (int j = 0; j < k; ++j)
              if ((sel[j] & 31) == lane) {
#pragma unroll
                for (int s = 0; s < kPerLane; ++s)
                  if ((sel[j] >> 5) == s) hist[s]++;
              }
          } else if (lane == 0) {
            for (int j = 0; j < k; ++j) atomicAdd(pred_counts + (size_t)(g - 1) * E + sel[j], 1);
          }
        }
      }
    }
  }
#pragma unroll
  for (int s = 0; s < kPerLane; ++s) {
    const int e = lane + 32 * s;
    if (e < E) {
      block_counts[(size_t)blk * E + e] = hist[s];
      if (hist[s]) atomicAdd(counts + e, hist[s]);
    }
  }
}

int gate_num_blocks(int T) { return (T + kBlockTokens - 1) / kBlockTokens; }

cudaError_t launch_gate_topk(const __nv_bfloat16* x, int T, int d, const __nv_bfloat16* w_all, int E,
                             int n_pred, int k, int32_t* ids, float* wts, int32_t* counts,
                             int32_t* block_counts, int32_t* pred_counts, cudaStream_t stream) {
  if (T <= 0) return cudaSuccess;
  if (E * (1 + n_pred) > 32 * kPerLane || k > 8 || (d % 8) != 0) return cudaErrorInvalidValue;
  const int nblk = gate_num_blocks(T);
  const dim3 grid((nblk + kWarpsPerCta - 1) / kWarpsPerCta), block(kWarpsPerCta * 32);
  const int Etot = E * (1 + n_pred);
  if (Etot <= 8)
    gate_topk_kernel<4, 8><<<grid, block, 0, stream>>>(x, T, d, w_all, E, n_pred, k, ids, wts, counts,
                                                        block_counts, pred_counts);
  else if (Etot <= 16)
    gate_topk_kernel<2, 16><<<grid, block, 0, stream>>>(x, T, d, w_all, E, n_pred, k, ids, wts, counts,
                                                         block_counts, pred_counts);
  else
    gate_topk_kernel<1, 32><<<grid, block, 0, stream>>>(x, T, d, w_all, E, n_pred, k, ids, wts, counts,
                                                         block_counts, pred_counts);
  return cudaGetLastError();
}

}  // namespace moe
