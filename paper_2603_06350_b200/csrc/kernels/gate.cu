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
// Work decomposition: one CTA (8 warps) owns a block of 32 consecutive tokens
// — the granularity of block_counts[], the stable prefix the dispatch kernel
// scans — and each warp owns TOKG of them.  A lane owns 8 contiguous columns
// per 256-column step, so x is read with 16-byte L1-bypassing loads (512 B
// coalesced per warp), unrolled so each lane keeps TOKG x kUnroll loads in
// flight; the gate rows (64 KB at d=4096, E=8) stay L1-resident and each
// 16-byte weight vector is reused for TOKG tokens.  Partial sums are
// all-reduced with xor shuffles; lane (e mod 32) keeps expert e for the
// warp arg-max.  The block histogram is built with shared-memory atomics and
// flushed with one global atomicAdd per (block, expert): the atomics-based
// per-expert load histogram.
//
// The predictor weights (n_pred target layers, each [E, d]) are stacked under
// the gate weights: the same pass over x yields pred_counts[p][E] (histogram
// only), so K2 costs no extra HBM read of x while E*(1+n_pred) <= EC.
#include <cfloat>
#include <cstdint>

#include "sm100_ptx.cuh"

namespace moe {

namespace {

constexpr int kBlockTokens = 32;  // tokens per CTA == per block_counts row
constexpr int kPerLane = 8;       // stacked experts per lane -> E*(1+n_pred) <= 256

// Top-k over the experts [base, base+E) of a stacked logit vector held as
// lane l -> stacked index l + 32 s.  Every lane returns the same ids/logits.
__device__ __forceinline__ void warp_topk(const float (&own)[kPerLane], int base, int E, int k,
                                          int (&ids_out)[8], float (&logit_out)[8]) {
  const int lane = lane_id();
  uint32_t taken = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    if (j >= k) break;
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
template <int TOKG, int EC, int kUnroll>
__global__ void __launch_bounds__(kBlockTokens / TOKG * 32)
gate_topk_kernel(const __nv_bfloat16* __restrict__ x, int T, int d,
                 const __nv_bfloat16* __restrict__ w_all, int E, int n_pred, int k,
                 int32_t* __restrict__ ids, float* __restrict__ wts, int32_t* __restrict__ counts,
                 int32_t* __restrict__ block_counts, int32_t* __restrict__ pred_counts) {
  constexpr int kWarps = kBlockTokens / TOKG;
  __shared__ int hist[kPerLane * 32];
  const int warp = threadIdx.x >> 5;
  const int lane = lane_id();
  const int blk = blockIdx.x;
  const int Etot = E * (1 + n_pred);
  for (int i = threadIdx.x; i < E; i += blockDim.x) hist[i] = 0;
  __syncthreads();

  const int t0 = blk * kBlockTokens + warp * TOKG;
  const int ntok = max(0, min(TOKG, T - t0));
  float own[TOKG][kPerLane];
#pragma unroll
  for (int q = 0; q < TOKG; ++q)
#pragma unroll
    for (int s = 0; s < kPerLane; ++s) own[q][s] = -FLT_MAX;

  if (ntok > 0) {
    for (int e0 = 0; e0 < Etot; e0 += EC) {
      float acc[TOKG][EC];
#pragma unroll
      for (int q = 0; q < TOKG; ++q)
#pragma unroll
        for (int c = 0; c < EC; ++c) acc[q][c] = 0.0f;

      for (int col0 = lane * 8; col0 < d; col0 += 256 * kUnroll) {
        int4 raw[kUnroll][TOKG];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
#pragma unroll
          for (int q = 0; q < TOKG; ++q) {
            const int col = col0 + 256 * u;
            raw[u][q] = (q < ntok && col < d) ? ld_nc_v4(x + (size_t)(t0 + q) * d + col) : make_int4(0, 0, 0, 0);
          }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const int col = col0 + 256 * u;
          if (col >= d) break;
          float xv[TOKG][8];
#pragma unroll
          for (int q = 0; q < TOKG; ++q) {
            const uint32_t* p = reinterpret_cast<const uint32_t*>(&raw[u][q]);
#pragma unroll
            for (int i = 0; i < 4; ++i) { xv[q][2 * i] = bf16lo(p[i]); xv[q][2 * i + 1] = bf16hi(p[i]); }
          }
#pragma unroll
          for (int c = 0; c < EC; ++c) {
            if (e0 + c < Etot) {
              const int4 wr = __ldg(reinterpret_cast<const int4*>(w_all + (size_t)(e0 + c) * d + col));
              const uint32_t* p = reinterpret_cast<const uint32_t*>(&wr);
              float wv[8];
#pragma unroll
              for (int i = 0; i < 4; ++i) { wv[2 * i] = bf16lo(p[i]); wv[2 * i + 1] = bf16hi(p[i]); }
#pragma unroll
              for (int q = 0; q < TOKG; ++q)
#pragma unroll
                for (int i = 0; i < 8; ++i) acc[q][c] = fmaf(xv[q][i], wv[i], acc[q][c]);
            }
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
          if (lane == 0) {
            if (g == 0) {
              float z = 0.0f, p[8];
#pragma unroll
              for (int j = 0; j < 8; ++j)
                if (j < k) { p[j] = expf(lg[j] - lg[0]); z += p[j]; }
#pragma unroll
              for (int j = 0; j < 8; ++j)
                if (j < k) {
                  ids[(size_t)t * k + j] = sel[j];
                  wts[(size_t)t * k + j] = p[j] / z;
                  atomicAdd(&hist[sel[j]], 1);
                }
            } else {
#pragma unroll
              for (int j = 0; j < 8; ++j)
                if (j < k) atomicAdd(pred_counts + (size_t)(g - 1) * E + sel[j], 1);
            }
          }
        }
      }
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    const int h = hist[e];
    block_counts[(size_t)blk * E + e] = h;
    if (h) atomicAdd(counts + e, h);
  }
}

int gate_num_blocks(int T) { return (T + kBlockTokens - 1) / kBlockTokens; }

cudaError_t launch_gate_topk(const __nv_bfloat16* x, int T, int d, const __nv_bfloat16* w_all, int E,
                             int n_pred, int k, int32_t* ids, float* wts, int32_t* counts,
                             int32_t* block_counts, int32_t* pred_counts, cudaStream_t stream) {
  if (T <= 0) return cudaSuccess;
  if (E * (1 + n_pred) > 32 * kPerLane || k > 8 || (d % 8) != 0) return cudaErrorInvalidValue;
  const int nblk = gate_num_blocks(T);
  const int Etot = E * (1 + n_pred);
  if (Etot <= 8)
    gate_topk_kernel<4, 8, 2><<<nblk, 256, 0, stream>>>(x, T, d, w_all, E, n_pred, k, ids, wts, counts,
                                                     block_counts, pred_counts);
  else if (Etot <= 16)
    gate_topk_kernel<2, 16, 4><<<nblk, 512, 0, stream>>>(x, T, d, w_all, E, n_pred, k, ids, wts, counts,
                                                      block_counts, pred_counts);
  else
    gate_topk_kernel<2, 16, 4><<<nblk, 512, 0, stream>>>(x, T, d, w_all, E, n_pred, k, ids, wts, counts,
                                                       block_counts, pred_counts);
  return cudaGetLastError();
}

}  // namespace moe
