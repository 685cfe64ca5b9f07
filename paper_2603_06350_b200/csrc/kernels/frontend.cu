// frontend.cu — the decode front end in ONE launch: K1 gate (+ K2 predictor)
// -> top-k -> K3 dispatch plan, ranking and row scatter, for a single GPU and
// small batches (up to 148 token blocks: cfg5's 256 tokens, cfg1's 2048).
//
// At decode the separate launches (split-K gate, gate finish, dispatch) each
// move a few hundred KB to a few MB, so each costs its launch latency, one
// kernel drain and a handful of dependent L2 round trips — ~25 us of a ~200 us
// layer (profiles/launches_cfg5_r02.csv) for ~10 MB of traffic.  Here one
// cooperative grid of nblk x splits CTAs (the gate's split-K grid, all
// co-resident) runs the three phases back to back, separated by two grid-wide
// barriers:
//
//   A  split-K partial logits of (32-token block, K split) -> L2 scratch
//      (block_partial_logits, the gate kernel's fragment mapping and ordered
//      K-slice sum).  (The decode weight prefetch stays on its side stream:
//      issued from here it delays this phase more than it saves in the GEMM,
//      profiles/ab_frontend_r02.md.)
//   B  token t on CTA t mod nctas, one warp: sums the splits' partial logits in
//      slice order (the finish kernel's arithmetic), top-k (lowest index wins
//      ties), softmax over the k, ids / weights; predictor slots add into their
//      histograms.
//   C  CTA (b, y): histograms from the ids (every CTA counts all T*k ids out
//      of L2, so no histogram atomics and no zeroing launch), the local plan
//      (one merged replica per expert, rows in expert order — the same plan
//      block_prefix_kernel / dispatch_kernel build), the stable rank of each of
//      block b's assignments, its row codes, and the scatter of column split y
//      of block b's rows into the permuted buffer.  CTA (0, 0) writes the plan,
//      the gate histogram and its host mirror, then the grid lets the GEMM
//      launch (PDL) while the rows are still being scattered.
//
// Same ids, weights, counts, row codes and plan as the three-kernel path
// (tests/test_gpu_frontend.py compares both with the oracle and each other).
#include <algorithm>
#include <atomic>
#include <cstdint>

#include <cooperative_groups.h>

#include "dispatch_plan.h"
#include "gate_common.cuh"
#include "sm100_ptx.cuh"

namespace moe {

namespace {

struct FrontArgs {
  const __nv_bfloat16* x;
  const __nv_bfloat16* w_all;  // [(1 + n_pred) * E, d]
  int32_t* ids;                // [T, k]
  float* wts;                  // [T, k]
  int32_t* counts;             // [E * (1 + n_pred)]: gate histogram, then predictor histograms
  int32_t* block_counts;       // [nblk, E]
  float* partial;              // [splits][nblk][32][8 NT] split-K scratch
  int32_t* host_counts;        // mapped pinned mirror of counts (nullptr: none)
  const float* pred_w2;        // predictor MLP W2 (nullptr: linear)
  uint32_t mlp_mask;
  int T, d, E, n_pred, k, splits;
  __nv_bfloat16* xp;           // permuted rows [T * k, d]
  uint32_t* row_code;          // [T, k]
  DevPlan* plan;
  const uint8_t* prefetch;     // first bytes of the GEMM's weights (nullptr: none)
  unsigned long long prefetch_bytes;
  unsigned long long* trace;   // MOE_FRONT_TRACE: per CTA 16 %globaltimer stamps at the phase edges (nullptr: off)
};

__device__ __forceinline__ void stamp(const FrontArgs& a, int cta, int i) {
  if (a.trace && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[cta * 16 + i] = t;
  }
}

// Grid-wide barrier: cooperative_groups' grid sync (the launch is
// cooperative).  Measured against a hand-rolled generation barrier (one
// 64-bit atomic word, the last arrival bumps the generation): 1.1-1.3 vs
// 1.6-2.1 us from the last arrival to the release at cfg5
// (profiles/ab_frontend_r02.md).
__device__ __forceinline__ void grid_barrier() { cooperative_groups::this_grid().sync(); }

template <int NT, bool MLP>
__global__ void __launch_bounds__(kWarps * 32, 1) frontend_kernel(const __grid_constant__ FrontArgs a) {
  constexpr int kCols = 8 * NT;
  constexpr int kLd = kCols + 4;
  constexpr int S = (kCols + 31) / 32;  // logits per lane in the top-k
  __shared__ float red[kBlockTokens * kLd];  // phase A partial sums; phase B per-warp rows
  __shared__ int s_cnt[kMaxExperts], s_pre[kMaxExperts], s_row[kMaxExperts];
  __shared__ uint32_t s_mask[kMaxExperts];
  __shared__ uint32_t codes[kBlockTokens * 8];
  const int warp = threadIdx.x >> 5, lane = lane_id();
  const int nblk = gridDim.x;
  const int nctas = gridDim.x * gridDim.y;
  const int cta = blockIdx.y * nblk + blockIdx.x;
  const int T = a.T, E = a.E, k = a.k;
  const int Etot = E * (1 + a.n_pred);

  // ---------------------------------------------------------------- phase A
  stamp(a, cta, 0);
  if (a.prefetch && threadIdx.x == 0) {
    // the GEMM streams the experts' weights in order: its first ~N MB go to L2
    // now, while this grid reads a few MB (256 KB pieces spread over the CTAs)
    constexpr unsigned long long kPiece = 256 * 1024;
    for (unsigned long long off = static_cast<unsigned long long>(cta) * kPiece; off < a.prefetch_bytes;
         off += static_cast<unsigned long long>(nctas) * kPiece) {
      const unsigned long long n = a.prefetch_bytes - off < kPiece ? a.prefetch_bytes - off : kPiece;
      bulk_prefetch_l2(a.prefetch + off, static_cast<uint32_t>(n & ~15ull));
    }
  }
  // the histograms accumulate atomically in phase B
  if (cta == 0)
    for (int i = threadIdx.x; i < Etot; i += blockDim.x) a.counts[i] = 0;
  if (blockIdx.y == 0)
    for (int e = threadIdx.x; e < E; e += blockDim.x) a.block_counts[(size_t)blockIdx.x * E + e] = 0;
  block_partial_logits<NT>(a.x, T, a.d, a.w_all, Etot, blockIdx.x, blockIdx.y, gridDim.y, red);
  {
    float* dst = a.partial + ((size_t)blockIdx.y * nblk + blockIdx.x) * kBlockTokens * kCols;
    for (int i = threadIdx.x; i < kBlockTokens * kCols; i += blockDim.x) dst[i] = red[(i / kCols) * kLd + i % kCols];
  }
  stamp(a, cta, 1);
  grid_barrier();
  stamp(a, cta, 3);

  // ---------------------------------------------------------------- phase B
  for (int t = warp * nctas + cta; t < T; t += kWarps * nctas) {
    const int blk = t / kBlockTokens, r = t % kBlockTokens;
    float* row = red + warp * kLd;  // this warp's summed logits
    {
      const float* src = a.partial + ((size_t)blk * kBlockTokens + r) * kCols;
      const size_t slice_stride = (size_t)nblk * kBlockTokens * kCols;
      constexpr int kMaxSplit = 16;
      float v[kMaxSplit][S];
#pragma unroll
      for (int s = 0; s < kMaxSplit; ++s)
#pragma unroll
        for (int q = 0; q < S; ++q) {
          const int col = lane + 32 * q;
          v[s][q] = s < a.splits && col < kCols ? __ldcg(src + s * slice_stride + col) : 0.0f;
        }
#pragma unroll
      for (int q = 0; q < S; ++q) {
        float acc = v[0][q];
#pragma unroll
        for (int s = 1; s < kMaxSplit; ++s)
          if (s < a.splits) acc += v[s][q];
        const int col = lane + 32 * q;
        if (col < kCols) row[col] = acc;
      }
    }
    if (t == cta) stamp(a, cta, 4);
    __syncwarp();
    for (int gi = 0; gi <= a.n_pred; ++gi) {
      int sel[8];
      float lg[8];
      if (MLP && gi > 0 && ((a.mlp_mask >> (gi - 1)) & 1u))
        mlp_scores_inplace<S>(row + gi * E, E, a.pred_w2 + (size_t)(gi - 1) * E * E);
      warp_topk<S>(row, gi * E, E, k, sel, lg);
      // every lane holds the same k winners: lane j writes slot j
      if (gi == 0) {
        float z = 0.0f, pj = 0.0f;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (j < k) {
            const float p = expf(lg[j] - lg[0]);
            z += p;
            if (j == lane) pj = p;
          }
        if (lane < k) {
          int id = sel[0];
#pragma unroll
          for (int j = 1; j < 8; ++j)
            if (j == lane) id = sel[j];
          a.ids[(size_t)t * k + lane] = id;
          a.wts[(size_t)t * k + lane] = pj / z;
          atomicAdd(a.counts + id, 1);
          atomicAdd(a.block_counts + (size_t)blk * E + id, 1);
        }
      } else if (lane < k) {
        int id = sel[0];
#pragma unroll
        for (int j = 1; j < 8; ++j)
          if (j == lane) id = sel[j];
        atomicAdd(a.counts + (size_t)gi * E + id, 1);
      }
    }
    __syncwarp();
  }
  // phase C's first round of row loads (x is an input: nothing to wait for)
  const int b = blockIdx.x;
  const int t_base = b * kBlockTokens;
  const int ntok = min(kBlockTokens, T - t_base);
  const int chunks_all = a.d / 8;
  const int per = (chunks_all + gridDim.y - 1) / gridDim.y;
  const int c_begin = blockIdx.y * per, c_end = min(chunks_all, c_begin + per);
  const int nch = max(0, c_end - c_begin);
  const int items = ntok * nch;
  constexpr int U = 4;
  int4 v0[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int it = threadIdx.x + u * blockDim.x;
    if (it < items) {
      const int tk = it / nch;
      v0[u] = ld_nc_v4(a.x + (size_t)(t_base + tk) * a.d + (size_t)(c_begin + it - tk * nch) * 8);
    }
  }
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    s_mask[e] = 0u;
    s_pre[e] = 0;
  }
  stamp(a, cta, 5);
  grid_barrier();
  stamp(a, cta, 7);

  // ---------------------------------------------------------------- phase C
  // one round of L2 loads: block b's ids (slot j on warp j), the expert
  // totals and block b's prefix (the histogram rows of the blocks before it)
  const int t = t_base + lane;
  const bool live = lane < ntok;
  const int my = warp < k && live ? __ldcg(a.ids + (size_t)t * k + warp) : -1;
  for (int e = threadIdx.x; e < E; e += blockDim.x) s_cnt[e] = __ldcg(a.counts + e);
  {
    // P threads per expert sum rows q, q + P, ... < b, 8 loads in flight each
    // (consecutive threads read consecutive experts of one row)
    const int P = max(1, static_cast<int>(blockDim.x) / E);
    for (int i = threadIdx.x; i < E * P; i += blockDim.x) {
      const int e = i % E, q = i / E;
      int pre = 0;
      for (int b0 = q; b0 < b; b0 += 8 * P) {
        int v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = b0 + u * P < b ? __ldcg(a.block_counts + (size_t)(b0 + u * P) * E + e) : 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) pre += v[u];
      }
      if (pre) atomicAdd(&s_pre[e], pre);
    }
  }
  if (my >= 0) atomicOr(&s_mask[my], 1u << lane);  // tokens of block b that chose expert e
  __syncthreads();
  stamp(a, cta, 8);
  const bool writer = cta == 0;
  if (warp == 0) {
    // local plan: expert e's rows start at sum_{e' < e} n_e' (merged replicas)
    int row_carry = 0, seg_carry = 0;
    for (int e0 = 0; e0 < E; e0 += 32) {
      const int e = e0 + lane;
      const int n = e < E ? s_cnt[e] : 0;
      int incl = n;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += v;
      }
      const uint32_t active = __ballot_sync(0xffffffffu, n > 0);
      const int row0 = row_carry + incl - n;
      if (e < E) {
        s_row[e] = row0;
        if (writer) {
          DevPlan* p = a.plan;
          p->n_e[e] = n;
          p->src_off[e] = 0;
          p->rep_base[e] = e;
          p->rep_row_base[e] = row0;
          p->rep_remote[e] = 0;
          if (n > 0) p->segs[seg_carry + __popc(active & ((1u << lane) - 1u))] = GemmSeg{row0, n, e, 0};
          if (a.host_counts) a.host_counts[e] = n;
        }
      }
      row_carry += __shfl_sync(0xffffffffu, incl, 31);
      seg_carry += __popc(active);
    }
    if (writer && lane == 0) {
      DevPlan* p = a.plan;
      p->E = E;
      p->R = E;
      p->G = 1;
      p->rank = 0;
      p->nseg = seg_carry;
      p->rows_local = row_carry;
      p->rows_send = 0;
      p->rep_base[E] = E;
    }
  }
  if (writer && a.host_counts)  // predictor histograms are complete (barrier 2)
    for (int i = E + threadIdx.x; i < Etot; i += blockDim.x) a.host_counts[i] = __ldcg(a.counts + i);
  __syncthreads();
  // the GEMM reads the segment list before its griddepcontrol.wait: every CTA
  // triggers after the plan writer's fence (dependents start once all have)
  if (writer) __threadfence();
  griddep_launch_dependents();
  stamp(a, cta, 9);

  // stable rank of (token, slot) = earlier tokens of the block with the same expert
  if (my >= 0) {
    const int gr = s_pre[my] + __popc(s_mask[my] & ((1u << lane) - 1u));
    const uint32_t code = static_cast<uint32_t>(s_row[my] + gr);
    codes[lane * k + warp] = code;
    if (blockIdx.y == 0) a.row_code[(size_t)t * k + warp] = code;
  }
  __syncthreads();
  // scatter: this CTA's 16-byte chunks [c_begin, c_end) of every row of block b
  for (int i0 = threadIdx.x; i0 < items; i0 += blockDim.x * U) {
    int4 v[U];
    int tok[U], ch[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int it = i0 + u * blockDim.x;
      tok[u] = it / nch;
      ch[u] = c_begin + (it - tok[u] * nch);
      if (i0 == threadIdx.x) v[u] = v0[u];  // first round: loaded before barrier 2
      else if (it < items) v[u] = ld_nc_v4(a.x + (size_t)(t_base + tok[u]) * a.d + (size_t)ch[u] * 8);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (i0 + u * blockDim.x >= items) break;
      for (int j = 0; j < k; ++j)
        st_v4(a.xp + (size_t)codes[tok[u] * k + j] * a.d + (size_t)ch[u] * 8, v[u]);
    }
  }
  __syncthreads();
  stamp(a, cta, 10);
}

}  // namespace

int gate_num_blocks(int T);
// The fused front end applies to single-GPU bf16 batches with <= 128 stacked
// logit columns whose split-K grid (token blocks x K splits) fits on the SMs at
// once: up to 148 blocks (4736 tokens; cfg5 8 x 16 CTAs, cfg1 64 x 2).
// K splits: the most (<= 16, a power of two) that keep the grid on the SMs
static int front_splits(int nblk, int d, int num_sms) {
  int s = 1;
  while (s < 16 && nblk * s * 2 <= num_sms && d % (kSlices * 32 * s * 2) == 0) s *= 2;
  return s;
}

bool frontend_applies(int T, int d, int Etot, int k, int num_sms) {
  if (T <= 0 || k < 1 || k > 8 || Etot > 128 || d % 256) return false;
  const int nblk = gate_num_blocks(T);
  return nblk <= num_sms && nblk * front_splits(nblk, d, num_sms) <= num_sms;
}

cudaError_t launch_frontend(const __nv_bfloat16* x, int T, int d, const __nv_bfloat16* w_all, int E, int n_pred, int k,
                            int32_t* ids, float* wts, int32_t* counts, int32_t* block_counts, float* partial,
                            int32_t* host_counts, const float* pred_w2, unsigned mlp_mask, __nv_bfloat16* xp,
                            uint32_t* row_code, DevPlan* plan, const void* prefetch, size_t prefetch_bytes,
                            unsigned long long* trace, cudaStream_t stream) {
  const int Etot = E * (1 + n_pred);
  const int nblk = gate_num_blocks(T);
  int sms = 148;
  {
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int splits = front_splits(nblk, d, sms);
  FrontArgs a{};
  a.x = x;
  a.w_all = w_all;
  a.ids = ids;
  a.wts = wts;
  a.counts = counts;
  a.block_counts = block_counts;
  a.partial = partial;
  a.host_counts = host_counts;
  a.pred_w2 = pred_w2;
  a.mlp_mask = mlp_mask;
  a.T = T;
  a.d = d;
  a.E = E;
  a.n_pred = n_pred;
  a.k = k;
  a.splits = splits;
  a.xp = xp;
  a.row_code = row_code;
  a.plan = plan;
  a.prefetch = static_cast<const uint8_t*>(prefetch);
  a.prefetch_bytes = prefetch ? prefetch_bytes : 0;
  a.trace = trace;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nblk, splits);
  cfg.blockDim = dim3(kWarps * 32);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // the grid barriers need every CTA resident
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const bool with_mlp = pred_w2 != nullptr && (mlp_mask & ((n_pred >= 32 ? 0u : (1u << n_pred)) - 1u)) != 0;
#define MOE_FRONT_CASE(NT_)                                                                 \
  if (Etot <= 8 * NT_) {                                                                    \
    if (with_mlp) return cudaLaunchKernelEx(&cfg, frontend_kernel<NT_, true>, a);           \
    return cudaLaunchKernelEx(&cfg, frontend_kernel<NT_, false>, a);                        \
  }
  MOE_FRONT_CASE(1)
  MOE_FRONT_CASE(2)
  MOE_FRONT_CASE(4)
  MOE_FRONT_CASE(8)
  MOE_FRONT_CASE(16)
#undef MOE_FRONT_CASE
  return cudaErrorInvalidValue;
}

cudaError_t preload_frontend_kernels() {
  cudaFuncAttributes fa;
  const void* fns[] = {
#define MOE_FRONT_FNS(NT_) \
  reinterpret_cast<const void*>(frontend_kernel<NT_, false>), reinterpret_cast<const void*>(frontend_kernel<NT_, true>)
      MOE_FRONT_FNS(1), MOE_FRONT_FNS(2), MOE_FRONT_FNS(4), MOE_FRONT_FNS(8), MOE_FRONT_FNS(16)};
#undef MOE_FRONT_FNS
  for (const void* f : fns) {
    cudaError_t e = cudaFuncGetAttributes(&fa, f);
    if (e != cudaSuccess) return e;
    // the same shared-memory carveout as the GEMM that follows (PDL): its CTAs
    // may then share an SM with this grid's CTAs without a reconfiguration
    e = cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace moe
