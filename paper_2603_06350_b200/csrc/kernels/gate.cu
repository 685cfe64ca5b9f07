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
// The op is an HBM-bound skinny GEMM (N = E*(1+n_pred) <= 256 logits per
// token); it uses the warp-level tensor-core MMA (m16n8k16, bf16 in, fp32
// accumulate) only so the FMA issue rate never limits the stream of x.
//
// Work decomposition: one CTA (8 warps) owns a block of 32 consecutive tokens
// — the granularity of block_counts[], the stable prefix the dispatch kernel
// scans.  Warp w takes m-tile (w & 1) (16 tokens) and K-slice (w >> 1), so a
// block keeps 8 independent 16-byte-load streams in flight.  Fragments are
// loaded straight from global memory: the 16 k-slots of one MMA are mapped to
// features so that lane (g, c) needs 4 CONSECUTIVE features of row g / row
// g+8 / expert g (slots 2c,2c+1 <-> f, f+1 and 2c+8,2c+9 <-> f+2, f+3,
// identical for A and B), i.e. one 16-byte load per row feeds two MMAs.
// K-slices are summed into shared memory in a fixed order (deterministic),
// then one warp per 4 tokens does the arg-max top-k, the softmax and the
// shared-memory histogram, flushed with one global atomicAdd per (block,
// expert) — the atomics-based per-expert histogram.
//
// Small batches (decode: 256 tokens = 8 blocks) split K over gridDim.y CTAs
// per block as well; each CTA publishes its partial logits and
// gate_finish_kernel sums the slices in order before the same top-k.
//
// Exactness: on the synthetic grid every partial sum is a
// multiple of 2^-16 below 2^6, so any fp32 summation order — the MMA's
// included — yields the exact logit, and ids match the CPU oracle bit for bit.
#include <algorithm>
#include <cfloat>
#include <atomic>
#include <cstdint>
#include <utility>

#include <cooperative_groups.h>
#include <cuda.h>

#include "gate_common.cuh"
#include "sm100_ptx.cuh"

namespace moe {

namespace {

// top-k, softmax and histograms for `ntok` tokens of one 32-token block,
// starting at token tok0 of the block, whose stacked logits sit in shared
// memory (row stride LD, row 0 = tok0); warp w handles ntok / kWarps tokens.
// ACCUM: the block's histogram row is shared with other CTAs (atomic adds
// into a zeroed row) instead of being written whole.
template <int LD, bool ACCUM, bool MLP, int BAR = 0>
__device__ __forceinline__ void select_and_count(const float* red, int* hist, int blk, int tok0, int ntok, int T,
                                                 int E, int n_pred, int k, int32_t* __restrict__ ids,
                                                 float* __restrict__ wts, int32_t* __restrict__ counts,
                                                 int32_t* __restrict__ block_counts,
                                                 int32_t* __restrict__ pred_counts, const PredictorMlp& mlp) {
  const int warp = threadIdx.x >> 5, lane = lane_id();
  constexpr int S = (LD - 4 + 31) / 32;  // E * (1 + n_pred) <= LD - 4 columns
  const int per = ntok / kWarps;
  for (int q = 0; q < per; ++q) {
    const int lt = warp * per + q;
    const int t = blk * kBlockTokens + tok0 + lt;
    if (t >= T) break;
    const float* row = red + lt * LD;
    for (int gi = 0; gi <= n_pred; ++gi) {
      int sel[8];
      float lg[8];
      if (MLP && gi > 0 && ((mlp.mask >> (gi - 1)) & 1u))
        mlp_scores_inplace<S>(const_cast<float*>(row) + gi * E, E, mlp.w2 + (size_t)(gi - 1) * E * E);
      warp_topk<S>(row, gi * E, E, k, sel, lg);
      if (lane == 0) {
        if (gi == 0) {
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
            if (j < k) atomicAdd(pred_counts + (size_t)(gi - 1) * E + sel[j], 1);
        }
      }
    }
  }
  // BAR = 0: the whole CTA; otherwise named barrier BAR over the kWarps consumer warps
  if (BAR == 0) __syncthreads(); else named_bar_sync(BAR, kWarps * 32);
  for (int e = threadIdx.x; e < E; e += kWarps * 32) {
    const int h = hist[e];
    if (ACCUM) {
      if (h) atomicAdd(block_counts + (size_t)blk * E + e, h);
    } else {
      block_counts[(size_t)blk * E + e] = h;
    }
    if (h) atomicAdd(counts + e, h);
  }
}

// Host mirror of the histograms (single GPU): the last CTA of the grid to
// finish copies counts[0, n) — gate then predictor histograms — into mapped
// pinned memory for the host planner, instead of a separate copy kernel.
struct CountsMirror {
  int32_t* host;      // mapped pinned [n]; nullptr = no mirror
  unsigned* ticket;   // CTAs done (self-resetting)
  int n;
};

__device__ __forceinline__ void publish_counts(const int32_t* counts, const CountsMirror& m, unsigned n_ctas) {
  if (!m.host) return;
  __shared__ bool last;
  __threadfence();  // this CTA's histogram atomics are visible device-wide
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(m.ticket, 1u) == n_ctas - 1;
  __syncthreads();
  if (last) {
    __threadfence();
    for (int i = threadIdx.x; i < m.n; i += blockDim.x) m.host[i] = __ldcg(counts + i);
    if (threadIdx.x == 0) *m.ticket = 0u;
  }
}

}  // namespace

// x [T, d] bf16; w_all [(1 + n_pred) * E, d] bf16 (rows 0..E-1 = gate).
// Outputs: ids [T, k] i32, weights [T, k] f32, counts [E] i32 (atomic; caller
// zeroes), block_counts [ceil(T/32), E] i32, pred_counts [n_pred, E] (atomic).
// NT = n-tiles of 8 stacked logits (E * (1 + n_pred) <= 8 * NT).  With
// gridDim.y > 1 the CTA covers a 1/gridDim.y share of d and writes its
// partial logits to `partial` instead of selecting — or, launched as clusters
// of gridDim.y CTAs (cluster_reduce), the y-rank-0 CTA of each cluster sums
// the other CTAs' partial logits out of their shared memory (DSMEM) in slice
// order, the finish kernel's arithmetic, and selects: no second launch and no
// round trip of the partials through global memory.
constexpr int kMaxClusterSplits = 8;

template <int NT, bool MLP>
__global__ void __launch_bounds__(kWarps * 32)
gate_topk_kernel(const __nv_bfloat16* __restrict__ x, int T, int d, const __nv_bfloat16* __restrict__ w_all, int E,
                 int n_pred, int k, int32_t* __restrict__ ids, float* __restrict__ wts, int32_t* __restrict__ counts,
                 int32_t* __restrict__ block_counts, int32_t* __restrict__ pred_counts, float* __restrict__ partial,
                 const __grid_constant__ CountsMirror mirror, const __grid_constant__ PredictorMlp mlp,
                 int cluster_reduce) {
  constexpr int kCols = 8 * NT;
  constexpr int kLd = kCols + 4;  // padded row of the reduction buffer
  __shared__ float red[kBlockTokens * kLd];
  __shared__ int hist[256];
  const int blk = blockIdx.x;
  const int Etot = E * (1 + n_pred);
  for (int i = threadIdx.x; i < E; i += blockDim.x) hist[i] = 0;

  block_partial_logits<NT>(x, T, d, w_all, Etot, blk, blockIdx.y, gridDim.y, red);
  if (gridDim.y > 1 && cluster_reduce) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();  // every slice's partial logits are in its CTA's shared memory
    if (blockIdx.y == 0) {
      const int S = gridDim.y;
      const float* peer[kMaxClusterSplits];
#pragma unroll
      for (int q = 1; q < kMaxClusterSplits; ++q) peer[q] = q < S ? cl.map_shared_rank(red, q) : red;
      for (int i = threadIdx.x; i < kBlockTokens * kLd; i += blockDim.x) {
        float v[kMaxClusterSplits];
#pragma unroll
        for (int q = 1; q < kMaxClusterSplits; ++q) v[q] = q < S ? peer[q][i] : 0.0f;  // all loads in flight
        float a = red[i];
#pragma unroll
        for (int q = 1; q < kMaxClusterSplits; ++q)
          if (q < S) a += v[q];
        red[i] = a;
      }
    }
    cl.sync();  // the peers' shared memory stays alive until it has been read
    if (blockIdx.y != 0) return;
    griddep_launch_dependents();
    select_and_count<kLd, false, MLP>(red, hist, blk, 0, kBlockTokens, T, E, n_pred, k, ids, wts, counts,
                                      block_counts, pred_counts, mlp);
    publish_counts(counts, mirror, gridDim.x);
    return;
  }
  if (gridDim.y > 1) {
    float* dst = partial + ((size_t)blockIdx.y * gridDim.x + blk) * kBlockTokens * kCols;
    for (int i = threadIdx.x; i < kBlockTokens * kCols; i += blockDim.x) dst[i] = red[(i / kCols) * kLd + i % kCols];
    // the finishing CTAs add into the block's histogram row
    if (blockIdx.y == 0)
      for (int e = threadIdx.x; e < E; e += blockDim.x) block_counts[(size_t)blk * E + e] = 0;
    return;
  }
  griddep_launch_dependents();  // the block-prefix launch may be scheduled (it waits for this grid)
  select_and_count<kLd, false, MLP>(red, hist, blk, 0, kBlockTokens, T, E, n_pred, k, ids, wts, counts, block_counts,
                               pred_counts, mlp);
  publish_counts(counts, mirror, gridDim.x * gridDim.y);
}

// Large batches (prefill): a persistent streaming gate.  One CTA per SM walks
// the 32-token blocks b = blockIdx.x, + gridDim.x, ...; a producer warp streams
// each block through a 4-stage shared-memory ring in K-chunks of 512 features
// (32 rows x 1 KB per stage = eight 32 x 64 TMA boxes with the 128-byte
// swizzle, so the consumers' 16-byte fragment loads are bank-conflict free),
// so ~128 KB per SM stay in flight — against the 1-2 us loaded HBM latency that is what
// the per-block kernel (3-4 blocks resident per SM, ~56 KB in flight, 3.46
// blocks per SM on average -> a 4-block tail) could not keep.  8 consumer warps
// = 2 m-tiles x 4 K-slices of 128 features per stage run the same m16n8k16
// MMAs on the same fragment mapping; at a block's end the K-slices are summed
// in order (deterministic) and the same top-k / softmax / histogram runs while
// the producer is already streaming the next block.
constexpr int kStreamK = 512;                      // features per stage
constexpr int kStreamBox = kBlockTokens * 128;     // one 32-row x 64-feature TMA box (4 KB)
constexpr int kStreamStages = 4;
constexpr int kStreamStageBytes = (kStreamK / 64) * kStreamBox;
constexpr int kStreamThreads = (kWarps + 1) * 32;  // + producer warp
constexpr int kStreamSmem = kStreamStages * kStreamStageBytes + 1024;  // + 1024-byte alignment slack

template <int NT, bool MLP>
__global__ void __launch_bounds__(kStreamThreads, 1)
gate_stream_kernel(const __grid_constant__ CUtensorMap tmx, int T, int d, const __nv_bfloat16* __restrict__ w_all, int E,
                   int n_pred, int k, int32_t* __restrict__ ids, float* __restrict__ wts, int32_t* __restrict__ counts,
                   int32_t* __restrict__ block_counts, int32_t* __restrict__ pred_counts,
                   const __grid_constant__ CountsMirror mirror, const __grid_constant__ PredictorMlp mlp) {
  constexpr int kCols = 8 * NT;
  constexpr int kLd = kCols + 4;
  extern __shared__ uint8_t stream_raw[];
  uint8_t* stream_smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(stream_raw) + 1023) & ~uintptr_t(1023));
  __shared__ float red[kBlockTokens * kLd];
  __shared__ int hist[256];
  __shared__ __align__(8) uint64_t full[kStreamStages], empty[kStreamStages];
  const int warp = threadIdx.x >> 5, lane = lane_id();
  const int nblk = (T + kBlockTokens - 1) / kBlockTokens;
  const int n_chunks = d / kStreamK;
  const int Etot = E * (1 + n_pred);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStreamStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], kWarps); }
    fence_barrier_init();
  }
  __syncthreads();
  griddep_launch_dependents();  // the block-prefix launch may be scheduled (it waits for this grid)

  if (warp == kWarps) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      tma_prefetch_desc(&tmx);
      int stage = 0;
      uint32_t phase = 0;
      for (int b = blockIdx.x; b < nblk; b += gridDim.x) {
        for (int ch = 0; ch < n_chunks; ++ch) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* dst = stream_smem + stage * kStreamStageBytes;
          mbar_arrive_expect_tx(&full[stage], kStreamStageBytes);  // rows past T are zero-filled
#pragma unroll
          for (int j = 0; j < kStreamK / 64; ++j)
            tma_load_2d(dst + j * kStreamBox, &tmx, &full[stage], ch * kStreamK + j * 64, b * kBlockTokens);
          if (++stage == kStreamStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else {
    // ----------------------------------------------------- consumers (8 warps)
    const int g = lane >> 2, c = lane & 3;
    const int mt = warp & 1, ks = warp >> 1;
    int stage = 0;
    uint32_t phase = 0;
    const int4 zero = make_int4(0, 0, 0, 0);
    for (int b = blockIdx.x; b < nblk; b += gridDim.x) {
      for (int i = threadIdx.x; i < E; i += kWarps * 32) hist[i] = 0;
      const int r0 = b * kBlockTokens + mt * 16 + g;
      const bool v0 = r0 < T, v1 = r0 + 8 < T;
      float acc[NT][4];
#pragma unroll
      for (int n = 0; n < NT; ++n) acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.0f;
      for (int ch = 0; ch < n_chunks; ++ch) {
        mbar_wait(&full[stage], phase);
        const uint8_t* base = stream_smem + stage * kStreamStageBytes;
        const int ra = mt * 16 + g, rb = ra + 8;  // rows of this lane's A fragments
#pragma unroll
        for (int q = 0; q < kStreamK / kSlices / 32; ++q) {
          const int fl = ks * (kStreamK / kSlices) + q * 32 + 8 * c;  // feature within the chunk
          const int f = ch * kStreamK + fl;
          // box fl / 64, 16-byte chunk (fl % 64) / 8 of the row, 128B-swizzled
          const uint8_t* box = base + (fl >> 6) * kStreamBox;
          const int chunk = (fl & 63) >> 3;
          const int4 a_lo = v0 ? *reinterpret_cast<const int4*>(box + ra * 128 + ((chunk ^ (ra & 7)) << 4)) : zero;
          const int4 a_hi = v1 ? *reinterpret_cast<const int4*>(box + rb * 128 + ((chunk ^ (rb & 7)) << 4)) : zero;
#pragma unroll
          for (int n = 0; n < NT; ++n) {
            const int e = n * 8 + g;
            const int4 bw = e < Etot ? __ldg(reinterpret_cast<const int4*>(w_all + (size_t)e * d + f)) : zero;
            mma_bf16_16816(acc[n], a_lo.x, a_hi.x, a_lo.y, a_hi.y, bw.x, bw.y);
            mma_bf16_16816(acc[n], a_lo.z, a_hi.z, a_lo.w, a_hi.w, bw.z, bw.w);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        if (++stage == kStreamStages) { stage = 0; phase ^= 1; }
      }
      // ordered K-slice reduction (consumers only: named barrier 1)
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
        named_bar_sync(1, kWarps * 32);
      }
      select_and_count<kLd, false, MLP, 1>(red, hist, b, 0, kBlockTokens, T, E, n_pred, k, ids, wts, counts,
                                           block_counts, pred_counts, mlp);
      named_bar_sync(1, kWarps * 32);  // red / hist are reused by the next block
    }
  }
  __syncthreads();
  publish_counts(counts, mirror, gridDim.x);
}

// Large batches (prefill), tensor-core gate: 128-token tiles of x stream
// through an 8-stage TMA ring (64-feature boxes, 128-byte swizzle, L2
// evict_first) beside the matching 64-feature slice of the stacked gate /
// predictor rows (N = Etot rounded up to 16 <= 32, L2 evict_last; the rows
// past Etot are the map's zero fill); one elected thread issues
// tcgen05.mma (M = 128 tokens, N, K = 16) x4 per stage into a double-buffered
// TMEM accumulator.  Four epilogue warps each own one 32-token block: a
// tcgen05.ld gives every thread its token's Etot logits, so top-k, softmax and
// the block histogram (ballots, one per expert) need no shared memory and no
// shuffles.  The per-block kernel above keeps ~56 KB per SM in flight through
// register-direct 16-byte loads; here ~160 KB per SM are in flight and x is
// read once in 64-feature rows.  Exactness as for the other gate kernels: on
// the synthetic grid every partial sum is exact in fp32, whatever the order.
std::atomic<int> g_gate_tc{1};      // env MOE_GATE_TC=0: prefill batches keep the per-block mma.sync gate
std::atomic<int> g_gate_tc_bks{2};  // env MOE_GATE_TC_BKS: 64-feature k-blocks per ring stage (1, 2, 4)
constexpr int kTcTile = 128;                              // tokens per tile (UMMA M)
constexpr uint32_t kTcXBytes = kTcTile * 64 * 2;          // 16 KB x box (64 features)
constexpr int kTcThreads = 192;                           // producer, MMA, 4 epilogue warps
constexpr uint32_t kTcRowLd = 33;                         // epilogue staging row (floats), conflict-free
constexpr uint32_t kTcRingBudget = 196 * 1024;
// NC accumulator columns (16 or 32 >= Etot); BKS 64-feature k-blocks per stage
// (adjacent k-blocks of a row are requested together: 128 B -> BKS x 128 B
// of each token row per DRAM visit)
template <int NC, int BKS>
struct TcCfg {
  static constexpr uint32_t kWBytes = NC * 64 * 2;
  static constexpr uint32_t kStage = BKS * (kTcXBytes + kWBytes);
  static constexpr int kStages = kTcRingBudget / kStage < 16 ? kTcRingBudget / kStage : 16;
  static constexpr uint32_t kSmem = kStages * kStage + 256 + 4 * 32 * kTcRowLd * 4 + 1024;
};
// One token's top-k over slot gi's E <= W logits: order keys packed with
// W - 1 - e in 64 bits, k arg-max rounds as log2(W)-deep trees (the max is the
// largest logit and, on ties, the lowest expert: warp_topk_vals' rule).  Slot
// 0 reads the TMEM registers directly; predictor slots (runtime offset gi * E)
// the token's shared-memory row.  Returns the chosen-expert mask.
template <int W>
__device__ __forceinline__ uint32_t tc_token_topk(const uint32_t (&r)[32], const float* row, int gi, int E, int k,
                                                  int (&sel)[8], float (&lg)[8]) {
  uint64_t key[W];
#pragma unroll
  for (int c = 0; c < W; ++c) {
    if (c >= E) {
      key[c] = 0ull;  // out of the race
      continue;
    }
    const float v = gi == 0 ? __uint_as_float(r[c]) : row[gi * E + c];
    key[c] = (static_cast<uint64_t>(logit_key(v)) << 32) | static_cast<uint32_t>(W - 1 - c);
  }
  uint32_t chosen = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    if (j >= k) break;
    uint64_t m[W / 2];
#pragma unroll
    for (int c = 0; c < W / 2; ++c) m[c] = key[2 * c] > key[2 * c + 1] ? key[2 * c] : key[2 * c + 1];
#pragma unroll
    for (int w = W / 4; w >= 1; w /= 2)
#pragma unroll
      for (int c = 0; c < w; ++c) m[c] = m[c] > m[c + w] ? m[c] : m[c + w];
    const int be = W - 1 - static_cast<int>(m[0] & 0xffffffffu);
    sel[j] = be;
    lg[j] = key_logit(static_cast<uint32_t>(m[0] >> 32));
    chosen |= 1u << be;
#pragma unroll
    for (int c = 0; c < W; ++c)
      if (c == be) key[c] = 0ull;
  }
  return chosen;
}

template <int NC, int BKS>
__global__ void __launch_bounds__(kTcThreads, 1)
gate_tc_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmw, int T, int d,
               int E, int n_pred, int k, int32_t* __restrict__ ids, float* __restrict__ wts,
               int32_t* __restrict__ counts, int32_t* __restrict__ block_counts, int32_t* __restrict__ pred_counts,
               const __grid_constant__ CountsMirror mirror, unsigned long long* __restrict__ trace) {
  extern __shared__ uint8_t tc_raw[];
  // MOE_FRONT_TRACE: %globaltimer stamps per CTA (start, prologue, first / last stage, epilogue, end)
  auto stamp = [&](int i) {
    if (trace) {
      unsigned long long v;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
      trace[blockIdx.x * 16 + i] = v;
    }
  };
  if (threadIdx.x == 0) stamp(0);
  auto cstamp = [&](int i) {
    if (trace) trace[blockIdx.x * 16 + i] = clock64();
  };
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(tc_raw) + 1023) & ~uintptr_t(1023));
  using C = TcCfg<NC, BKS>;
  constexpr int kTcStages = C::kStages;
  constexpr uint32_t kTcStageBytes = C::kStage;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kTcStages * kTcStageBytes);
  uint64_t* empty = full + kTcStages;
  uint64_t* tfull = empty + kTcStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* rows = reinterpret_cast<float*>(smem + kTcStages * kTcStageBytes + 256);  // [4 warps][32][kTcRowLd]
  __shared__ int s_hist[32];  // this CTA's gate + predictor histograms (Etot <= 32)
  if (threadIdx.x < 32) s_hist[threadIdx.x] = 0;
  const int warp = threadIdx.x >> 5, lane = lane_id();
  const int n_tiles = (T + kTcTile - 1) / kTcTile;
  const int num_kb = d / (64 * BKS);  // stages per tile
  // this CTA's stages: (tile, k-stage) pairs i = 0 .. n_mine * num_kb - 1
  const int n_mine = blockIdx.x < n_tiles ? (n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int pre = min(kTcStages, n_mine * num_kb);  // issued before the CTA-wide sync
  auto issue = [&](int i, int stage, uint64_t pol_x, uint64_t pol_w) {
    const int t = blockIdx.x + (i / num_kb) * gridDim.x, kb = i % num_kb;
    uint8_t* st = smem + stage * kTcStageBytes;
    mbar_arrive_expect_tx(&full[stage], kTcStageBytes);  // OOB rows are zero-filled
#pragma unroll
    for (int q = 0; q < BKS; ++q)
      tma_load_2d_hint(st + q * kTcXBytes, &tmx, &full[stage], (kb * BKS + q) * 64, t * kTcTile, pol_x);
#pragma unroll
    for (int q = 0; q < BKS; ++q)
      tma_load_2d_hint(st + BKS * kTcXBytes + q * C::kWBytes, &tmw, &full[stage], (kb * BKS + q) * 64, 0, pol_w);
  };
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmx);
    tma_prefetch_desc(&tmw);
    for (int s = 0; s < kTcStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 4); }
    fence_barrier_init();
    // the first stages go out before TMEM allocation and the CTA sync (fresh
    // stages need no empty wait): the first HBM round trip starts at once
    const uint64_t pol_x = policy_evict_first(), pol_w = policy_evict_last();
    for (int i = 0; i < pre; ++i) issue(i, i, pol_x, pol_w);
  }
  if (warp == 1) tmem_alloc<64>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_launch_dependents();  // the block-prefix launch may be scheduled (it waits for this grid)
  if (threadIdx.x == 0) stamp(1);

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_x = policy_evict_first(), pol_w = policy_evict_last();
      int stage = pre % kTcStages;
      uint32_t phase = pre == kTcStages ? 1u : 0u;
      for (int i = pre; i < n_mine * num_kb; ++i) {
        mbar_wait(&empty[stage], phase ^ 1);
        issue(i, stage, pol_x, pol_w);
        if (++stage == kTcStages) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      constexpr uint32_t idesc = umma_idesc_bf16(kTcTile, NC);
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0;
      const uint32_t base = smem_u32(smem);
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t dcol = tmem_base + acc * 32;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (kb == 0) stamp(2);
          if (kb == num_kb - 1) stamp(3);
#pragma unroll
          for (int b = 0; b < BKS; ++b) {
            const uint64_t xa = umma_desc_sw128(base + stage * kTcStageBytes + b * kTcXBytes);
            const uint64_t wb = umma_desc_sw128(base + stage * kTcStageBytes + BKS * kTcXBytes + b * C::kWBytes);
#pragma unroll
            for (int q = 0; q < 4; ++q)
              tc_mma_bf16(dcol, xa + 2 * q, wb + 2 * q, idesc, (kb | b | q) != 0 ? 1u : 0u);
          }
          tc_commit(&empty[stage]);
          if (++stage == kTcStages) { stage = 0; phase ^= 1; }
        }
        tc_commit(&tfull[acc]);
        stamp(9);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    // epilogue: warp w owns TMEM lanes 32 (w % 4) .. + 31 = one 32-token block of the tile
    const int quarter = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      if (warp == 2 && lane == 0) stamp(6);
      uint32_t r[32];
      tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + acc * 32, r);
      tc_wait_ld();
      if (warp == 2 && lane == 0) { stamp(7); cstamp(13); }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      const int blk = tile * (kTcTile / kBlockTokens) + quarter;
      const int t = blk * kBlockTokens + lane;
      const bool live = t < T;
      // Slot gi's E logits -> NC order keys in registers (gi = 0 straight from
      // the TMEM load; predictor slots through a private shared-memory row, as
      // their offset gi * E is a runtime value), then k arg-max rounds as
      // log2(NC)-deep trees over (key, NC - 1 - e) packed in 64 bits: the max
      // is the largest logit and, on ties, the lowest expert (warp_topk_vals'
      // rule).  The serial 32-step scan this replaces was a dependent chain of
      // ~2.5k cycles per tile at the end of every CTA.
      float* row = rows + (quarter * 32 + lane) * kTcRowLd;
      if (n_pred > 0) {
#pragma unroll
        for (int c = 0; c < NC; ++c) row[c] = __uint_as_float(r[c]);
      }
      for (int gi = 0; gi <= n_pred; ++gi) {
        int sel[8];
        float lg[8];
        uint32_t chosen;  // bit e: this token chose expert e
        if (E <= 8)
          chosen = tc_token_topk<8>(r, row, gi, E, k, sel, lg);
        else
          chosen = tc_token_topk<NC>(r, row, gi, E, k, sel, lg);
        if (!live) chosen = 0u;
        if (warp == 2 && lane == 0 && gi == 0) { stamp(11); cstamp(14); }
        if (gi == 0 && live) {
          float z = 0.0f, p[8];
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (j < k) { p[j] = expf(lg[j] - lg[0]); z += p[j]; }
          if (k == 2) {  // the Mixtral / Phi shapes: one 8-byte store each
            reinterpret_cast<int2*>(ids)[t] = make_int2(sel[0], sel[1]);
            reinterpret_cast<float2*>(wts)[t] = make_float2(p[0] / z, p[1] / z);
          } else {
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (j < k) {
                ids[(size_t)t * k + j] = sel[j];
                wts[(size_t)t * k + j] = p[j] / z;
              }
          }
        }
        if (warp == 2 && lane == 0 && gi == 0) { stamp(12); cstamp(15); }
        // the block's histogram: one ballot per expert, lane e publishes expert e
        int mine = 0;
#pragma unroll
        for (int e = 0; e < NC; ++e) {
          if (e >= E) break;
          const int c = __popc(__ballot_sync(0xffffffffu, (chosen >> e) & 1u));
          if (lane == e) mine = c;
        }
        if (gi == 0 && lane < E && blk * kBlockTokens < T) block_counts[(size_t)blk * E + lane] = mine;
        if (lane < E && mine) atomicAdd(&s_hist[gi * E + lane], mine);  // one global add per CTA and slot
      }
      if (warp == 2 && lane == 0) stamp(8);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < E * (1 + n_pred) && s_hist[threadIdx.x])
    atomicAdd(threadIdx.x < E ? counts + threadIdx.x : pred_counts + (threadIdx.x - E), s_hist[threadIdx.x]);
  if (threadIdx.x == 0) stamp(4);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<64>(tmem_base);
  }
  publish_counts(counts, mirror, gridDim.x);
  if (threadIdx.x == 0) stamp(5);
}

bool gate_tc_applies(int T, int d, int Etot, int k, bool mlp) {
  return g_gate_tc.load(std::memory_order_relaxed) != 0 && T >= 64 * kTcTile && d % 256 == 0 && Etot <= 32 &&
         k <= 8 && !mlp;
}

cudaError_t launch_gate_tc(const CUtensorMap* tmx, const CUtensorMap* tmw, int T, int d, int E, int n_pred, int k,
                           int32_t* ids, float* wts, int32_t* counts, int32_t* block_counts, int32_t* pred_counts,
                           int32_t* host_counts, int host_n, unsigned* ticket, int num_sms, cudaStream_t stream,
                           unsigned long long* trace) {
  const CountsMirror mirror{host_counts, ticket, host_n};
  const int Etot = E * (1 + n_pred);
  const int tiles = (T + kTcTile - 1) / kTcTile;
  const int grid = tiles < num_sms ? tiles : num_sms;
  const int bks = g_gate_tc_bks.load(std::memory_order_relaxed);
#define MOE_TC_LAUNCH(NC_, BKS_)                                                                              \
  gate_tc_kernel<NC_, BKS_><<<grid, kTcThreads, TcCfg<NC_, BKS_>::kSmem, stream>>>(                           \
      *tmx, *tmw, T, d, E, n_pred, k, ids, wts, counts, block_counts, pred_counts, mirror, trace)
  if (Etot <= 16) {
    if (bks == 4) MOE_TC_LAUNCH(16, 4); else if (bks == 2) MOE_TC_LAUNCH(16, 2); else MOE_TC_LAUNCH(16, 1);
  } else {
    if (bks == 4) MOE_TC_LAUNCH(32, 4); else if (bks == 2) MOE_TC_LAUNCH(32, 2); else MOE_TC_LAUNCH(32, 1);
  }
#undef MOE_TC_LAUNCH
  return cudaGetLastError();
}

// Sums the split-K partial logits of kFinishTokens tokens of one 32-token
// block in slice order (deterministic; all slices are loaded before the
// first add, so the sum costs one memory latency, not `splits`), then top-k /
// softmax / histograms as in the fused kernel, one token per warp.
constexpr int kFinishTokens = kWarps;
constexpr int kMaxSplits = 16;

template <int NT, bool MLP>
__global__ void __launch_bounds__(kWarps * 32)
gate_finish_kernel(const float* __restrict__ partial, int splits, int T, int E, int n_pred, int k,
                   int32_t* __restrict__ ids, float* __restrict__ wts, int32_t* __restrict__ counts,
                   int32_t* __restrict__ block_counts, int32_t* __restrict__ pred_counts,
                   const __grid_constant__ CountsMirror mirror, const __grid_constant__ PredictorMlp mlp) {
  constexpr int kCols = 8 * NT;
  constexpr int kLd = kCols + 4;
  __shared__ float red[kFinishTokens * kLd];
  __shared__ int hist[256];
  const int blk = blockIdx.x, tok0 = blockIdx.y * kFinishTokens;
  const int nblk = gridDim.x;
  for (int i = threadIdx.x; i < E; i += blockDim.x) hist[i] = 0;
  for (int i = threadIdx.x; i < kFinishTokens * kCols; i += blockDim.x) {
    const float* src = partial + ((size_t)blk * kBlockTokens + tok0) * kCols + i;
    const size_t slice_stride = (size_t)nblk * kBlockTokens * kCols;
    float v[kMaxSplits];
#pragma unroll
    for (int s = 0; s < kMaxSplits; ++s) v[s] = s < splits ? __ldcg(src + s * slice_stride) : 0.0f;
    float acc = v[0];
#pragma unroll
    for (int s = 1; s < kMaxSplits; ++s)
      if (s < splits) acc += v[s];
    red[(i / kCols) * kLd + i % kCols] = acc;
  }
  __syncthreads();
  griddep_launch_dependents();
  select_and_count<kLd, true, MLP>(red, hist, blk, tok0, kFinishTokens, T, E, n_pred, k, ids, wts, counts, block_counts,
                              pred_counts, mlp);
  publish_counts(counts, mirror, gridDim.x * gridDim.y);
}

// Caller-given routing (moe_layer_forward_ids — the SURVEY §8 c3 bridge: ids
// replayed from the reference's route_tokens stream, workload.cpp:188-230,
// enter the data path here instead of K1).  One CTA per 32-token block, one
// thread per (token, slot): checks 0 <= id < E and that a token names each
// expert once (route_tokens rejects duplicates, workload.cpp:221-226), copies
// ids and weights (NULL weights: 1/k each) into the context's buffers, and
// writes the same block histogram row + global histogram the gate writes, so
// block prefix / dispatch / K4 / combine run unchanged.  A bad token is
// replaced by experts 0..k-1 with weight 0 (memory-safe downstream) and
// reported through *err = 1 + first bad token (the host raises MOE_EINVAL).
__global__ void __launch_bounds__(256)
route_ids_kernel(const int32_t* __restrict__ ids_in, const float* __restrict__ w_in, int T, int E, int k,
                 int32_t* __restrict__ ids, float* __restrict__ wts, int32_t* __restrict__ counts,
                 int32_t* __restrict__ block_counts, int* __restrict__ err) {
  __shared__ int hist[kMaxHistExperts];
  __shared__ unsigned char bad[kBlockTokens];
  const int blk = blockIdx.x;
  for (int i = threadIdx.x; i < E; i += blockDim.x) hist[i] = 0;
  if (threadIdx.x < kBlockTokens) bad[threadIdx.x] = 0;
  __syncthreads();
  const int lt = threadIdx.x / k, j = threadIdx.x % k;
  const int t = blk * kBlockTokens + lt;
  const bool live = lt < kBlockTokens && t < T;
  int id = 0;
  if (live) {
    id = __ldg(ids_in + (size_t)t * k + j);
    bool ok = id >= 0 && id < E;
    for (int q = 0; q < j; ++q) ok = ok && __ldg(ids_in + (size_t)t * k + q) != id;
    if (!ok) bad[lt] = 1;
  }
  __syncthreads();
  if (live) {
    float w = w_in ? __ldg(w_in + (size_t)t * k + j) : 1.0f / static_cast<float>(k);
    if (bad[lt]) {
      id = j;
      w = 0.0f;
      if (j == 0) atomicCAS(err, 0, 1 + t);
    }
    ids[(size_t)t * k + j] = id;
    wts[(size_t)t * k + j] = w;
    atomicAdd(&hist[id], 1);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    const int h = hist[e];
    block_counts[(size_t)blk * E + e] = h;
    if (h) atomicAdd(counts + e, h);
  }
}

cudaError_t launch_route_ids(const int32_t* ids_in, const float* w_in, int T, int E, int k, int32_t* ids, float* wts,
                             int32_t* counts, int32_t* block_counts, int* err, cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  if (k < 1 || k > 8 || k > E || E > kMaxHistExperts) return cudaErrorInvalidValue;
  route_ids_kernel<<<(T + kBlockTokens - 1) / kBlockTokens, 256, 0, s>>>(ids_in, w_in, T, E, k, ids, wts, counts, block_counts, err);
  return cudaGetLastError();
}

int gate_num_blocks(int T) { return (T + kBlockTokens - 1) / kBlockTokens; }

// K-splits for a batch: enough CTAs to cover the SMs twice, d/(4 S) a
// multiple of 32, at most 16.
std::atomic<int> g_gate_max_splits{16};  // env MOE_GATE_MAX_SPLITS (A/B); set at ctx creation
std::atomic<int> g_gate_cluster{0};      // env MOE_GATE_CLUSTER: 1 = split-K reduced inside a cluster (DSMEM), 0 = finish kernel (default: profiles/ab_gate_cluster_r02.md)
std::atomic<int> g_gate_min_splits{1};   // env MOE_GATE_MIN_SPLITS: split large batches too (A/B)
std::atomic<int> g_gate_stream{0};       // env MOE_GATE_STREAM=1: the persistent streaming gate for large batches (opt-in: 47 vs 39 us at cfg2, profiles/ab_gate_stream_r02.md)

int gate_splits(int T, int d) {
  const int nblk = gate_num_blocks(T);
  int s = 1;
  // the finish kernel sums at most kMaxSplits slices, a cluster holds at most
  // kMaxClusterSplits (portable cluster size): never split further
  const int cap = g_gate_cluster.load(std::memory_order_relaxed) ? kMaxClusterSplits : kMaxSplits;
  const int max_s = std::min(g_gate_max_splits.load(std::memory_order_relaxed), cap);
  while (s < max_s && nblk * s * 2 <= 2 * 148 && d % (kSlices * 32 * s * 2) == 0) s *= 2;
  const int min_s = g_gate_min_splits.load(std::memory_order_relaxed);
  while (s < min_s && s * 2 <= max_s && d % (kSlices * 32 * s * 2) == 0) s *= 2;
  return s;
}

// floats of split-K scratch a launch with these sizes needs
size_t gate_partial_floats(int T, int d, int Etot) {
  const int s = gate_splits(T, d);
  int nt = 1;
  while (8 * nt < Etot) nt *= 2;
  return s > 1 ? static_cast<size_t>(s) * gate_num_blocks(T) * kBlockTokens * 8 * nt : 0;
}

cudaError_t launch_gate_topk(const __nv_bfloat16* x, int T, int d, const __nv_bfloat16* w_all, int E,
                             int n_pred, int k, int32_t* ids, float* wts, int32_t* counts,
                             int32_t* block_counts, int32_t* pred_counts, float* partial, cudaStream_t stream,
                             int32_t* host_counts, int host_n, unsigned* ticket, const float* pred_w2,
                             unsigned mlp_mask, const CUtensorMap* tmx) {
  if (T <= 0) return cudaSuccess;
  const CountsMirror mirror{host_counts, ticket, host_n};
  const PredictorMlp mlp{pred_w2, mlp_mask};
  const int Etot = E * (1 + n_pred);
  if (Etot > 32 * kPerLane || k > 8 || (d % 256) != 0) return cudaErrorInvalidValue;
  const int nblk = gate_num_blocks(T);
  const int splits = partial ? gate_splits(T, d) : 1;
  const dim3 grid(nblk, splits), block(kWarps * 32);
  const bool with_mlp = pred_w2 != nullptr && (mlp_mask & ((n_pred >= 32 ? 0u : (1u << n_pred)) - 1u)) != 0;
  const bool in_cluster = splits > 1 && g_gate_cluster.load(std::memory_order_relaxed) != 0;
  // prefill: the persistent streaming gate (one CTA per SM, 4-stage ring)
  const bool stream_gate = tmx != nullptr && splits == 1 && nblk >= 148 && d % kStreamK == 0 && Etot <= 32 &&
                           g_gate_stream.load(std::memory_order_relaxed) != 0;
  const int stream_grid = nblk < 148 ? nblk : 148;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = splits;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = in_cluster ? 1 : 0;
#define MOE_GATE_LAUNCH(NT_, MLP_)                                                                          \
  {                                                                                                         \
    if (stream_gate) {                                                                                      \
      if constexpr (NT_ <= 4) {                                                                             \
        gate_stream_kernel<NT_, MLP_><<<stream_grid, kStreamThreads, kStreamSmem,                           \
                                        stream>>>(*tmx, T, d, w_all, E, n_pred, k, ids, wts, counts,        \
                                                  block_counts, pred_counts, mirror, mlp);                  \
        return cudaGetLastError();                                                                          \
      }                                                                                                     \
    }                                                                                                       \
    if (in_cluster)                                                                                         \
      return cudaLaunchKernelEx(&cfg, gate_topk_kernel<NT_, MLP_>, x, T, d, w_all, E, n_pred, k, ids, wts,  \
                                counts, block_counts, pred_counts, partial, mirror, mlp, 1);               \
    gate_topk_kernel<NT_, MLP_><<<grid, block, 0, stream>>>(x, T, d, w_all, E, n_pred, k, ids, wts, counts, \
                                                            block_counts, pred_counts, partial,            \
                                                            splits > 1 ? CountsMirror{} : mirror, mlp, 0); \
    if (splits > 1)                                                                                         \
      gate_finish_kernel<NT_, MLP_><<<dim3(nblk, kBlockTokens / kFinishTokens), block, 0, stream>>>(        \
          partial, splits, T, E, n_pred, k, ids, wts, counts, block_counts, pred_counts, mirror, mlp);      \
    return cudaGetLastError();                                                                              \
  }
#define MOE_GATE_CASE(NT_)                                                                                  \
  if (Etot <= 8 * NT_) {                                                                                    \
    if (with_mlp) MOE_GATE_LAUNCH(NT_, true)                                                                \
    MOE_GATE_LAUNCH(NT_, false)                                                                             \
  }
  MOE_GATE_CASE(1)
  MOE_GATE_CASE(2)
  MOE_GATE_CASE(4)
  MOE_GATE_CASE(8)
  MOE_GATE_CASE(16)
  MOE_GATE_CASE(32)
#undef MOE_GATE_LAUNCH
#undef MOE_GATE_CASE
  return cudaErrorInvalidValue;
}

// Load every kernel of this file now (CUDA 12 loads kernels lazily on first
// launch, and a lazy load may wait for the whole context — including a
// peer-exchange kernel spinning on another rank that shares the context).
cudaError_t preload_gate_kernels() {
  // the streaming gate's ring is dynamic shared memory beyond 48 KB (per device)
  const void* stream_fns[] = {
#define MOE_STREAM_FNS(NT_) \
  reinterpret_cast<const void*>(gate_stream_kernel<NT_, false>), reinterpret_cast<const void*>(gate_stream_kernel<NT_, true>)
      MOE_STREAM_FNS(1), MOE_STREAM_FNS(2), MOE_STREAM_FNS(4)};
#undef MOE_STREAM_FNS
  const std::pair<const void*, uint32_t> tc_fns[] = {
#define MOE_TC_FN(NC_, BKS_) {reinterpret_cast<const void*>(gate_tc_kernel<NC_, BKS_>), TcCfg<NC_, BKS_>::kSmem}
      MOE_TC_FN(16, 1), MOE_TC_FN(16, 2), MOE_TC_FN(16, 4), MOE_TC_FN(32, 1), MOE_TC_FN(32, 2), MOE_TC_FN(32, 4)};
#undef MOE_TC_FN
  for (const auto& f : tc_fns) {
    const cudaError_t e = cudaFuncSetAttribute(f.first, cudaFuncAttributeMaxDynamicSharedMemorySize, f.second);
    if (e != cudaSuccess) return e;
  }
  for (const void* f : stream_fns) {
    const cudaError_t e =
        cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, kStreamSmem);
    if (e != cudaSuccess) return e;
  }
  cudaFuncAttributes a;
  const void* fns[] = {
#define MOE_GATE_FNS(NT_)                                                                               \
  reinterpret_cast<const void*>(gate_topk_kernel<NT_, false>),                                          \
      reinterpret_cast<const void*>(gate_topk_kernel<NT_, true>),                                       \
      reinterpret_cast<const void*>(gate_finish_kernel<NT_, false>),                                    \
      reinterpret_cast<const void*>(gate_finish_kernel<NT_, true>)
      MOE_GATE_FNS(1), MOE_GATE_FNS(2), MOE_GATE_FNS(4), MOE_GATE_FNS(8), MOE_GATE_FNS(16), MOE_GATE_FNS(32)};
#undef MOE_GATE_FNS
  for (const void* f : fns) {
    const cudaError_t e = cudaFuncGetAttributes(&a, f);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace moe
