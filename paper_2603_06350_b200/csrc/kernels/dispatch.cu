// dispatch.cu — K3: replica-aware token dispatch, and K5: weighted top-k
// combine / unpermute.
//
// The reference's dispatcher is the rational rule "each replica of expert e
// carries actual[e] / R_e tokens" (proj/src/cost_model.cpp:98-106).  The real
// dispatcher makes it integer: the n_e assignments of expert
// e, in global (source rank, token) order, are cut into R_e contiguous ranges,
// replica r taking floor(n_e/R_e) + [r < n_e mod R_e].  Each rank lays out
// the rows it receives as segments in (expert, ordinal) order; within a
// segment, rows keep the global order, so the permutation is stable and
// bit-reproducible (no atomics decide positions).
//
// Pipeline (all on device, no host round trip once the plan is uploaded):
//   block_prefix_kernel  exclusive scan of the gate's per-32-token-block
//                        histograms -> each block's per-expert start rank.
//   dispatch_kernel      one CTA per 32-token block (x gridDim.y column
//                        splits for small batches): warp 0 ranks the block's
//                        (token, slot) assignments from per-expert token
//                        bitmasks (shared-memory atomicOr + popc), maps global
//                        rank -> replica -> destination row, and records a
//                        32-bit row code per assignment (target << 28 | row:
//                        local rows, the NCCL send buffer, or a peer's
//                        received rows); then all 4 warps stream the rows
//                        once from HBM and store each k times (128-bit).
//   combine_kernel       y_t = sum_j w_tj * Y[row(t, j)], fp32 accumulate in
//                        slot order, bf16 out; one warp per token.
#include <algorithm>
#include <cstdint>
#include <utility>

#include "dispatch_plan.h"
#include "sm100_ptx.cuh"

namespace moe {

// ------------------------------------------------------- block prefix scan
// block_pre[b][e] = src_off[e] + sum_{b' < b} block_counts[b'][e].  One CTA per
// expert column; each thread scans a contiguous chunk of blocks.
__device__ void plan_local_body(const int32_t* __restrict__ counts, int E, DevPlan* __restrict__ plan);

// local_counts != nullptr (single GPU): the dispatch plan is built by one extra
// CTA (index E) from the gate histogram, and every source offset is 0 — the
// plan kernel and the scan share one launch.
__global__ void __launch_bounds__(512)
block_prefix_kernel(const int32_t* __restrict__ block_counts, int nblk, int E,
                    const DevPlan* __restrict__ plan, int32_t* __restrict__ block_pre,
                    const int32_t* __restrict__ local_counts, DevPlan* __restrict__ local_plan) {
  griddep_wait();  // launched programmatically behind the gate
  const int e = blockIdx.x;
  if (e == E) {
    // the plan CTA lets dependents start only once the plan is written: with
    // T == 0 no dispatch runs, and GEMM1 (PDL) reads the segment list early
    plan_local_body(local_counts, E, local_plan);
    __threadfence();
    __syncthreads();
    griddep_launch_dependents();
    return;
  }
  griddep_launch_dependents();  // dispatch CTAs may be scheduled now (they wait for this grid)
  const int tid = threadIdx.x;
  const int per = (nblk + blockDim.x - 1) / blockDim.x;
  const int b0 = tid * per, b1 = min(nblk, b0 + per);
  int local = 0;
  for (int b = b0; b < b1; ++b) local += block_counts[(size_t)b * E + e];
  // exclusive scan of `local` across the CTA
  __shared__ int warp_sums[16];
  const int lane = tid & 31, warp = tid >> 5;
  int incl = local;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += v;
  }
  if (lane == 31) warp_sums[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int w = lane < (int)(blockDim.x >> 5) ? warp_sums[lane] : 0;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, w, off);
      if (lane >= off) w += v;
    }
    if (lane < (int)(blockDim.x >> 5)) warp_sums[lane] = w;  // inclusive warp prefix
  }
  __syncthreads();
  int run = (local_counts ? 0 : plan->src_off[e]) + (warp > 0 ? warp_sums[warp - 1] : 0) + incl - local;
  for (int b = b0; b < b1; ++b) {
    block_pre[(size_t)b * E + e] = run;
    run += block_counts[(size_t)b * E + e];
  }
}

// ------------------------------------------------------------- dispatch
// Single GPU with few 32-token blocks (decode): the dispatch CTAs build their
// own prefix row and the local plan from the gate's histograms, so the
// block-prefix launch disappears.  Every CTA sums block_counts[b' < b] for its
// block and scans the expert totals (one warp, 32 experts per step); CTA
// (0, 0) also writes the DevPlan the GEMMs read after their griddepcontrol.wait
// on this grid.  Same rows, same codes as block_prefix_kernel + plan_local_body.
struct LocalPlan {
  const int32_t* counts;        // [E] gate histogram; nullptr: read block_pre / plan as usual
  const int32_t* block_counts;  // [nblk][E]
  DevPlan* out;                 // written by CTA (0, 0)
};
constexpr int kFusedPlanMaxBlocks = 32;

template <int K>
__global__ void __launch_bounds__(128)
dispatch_kernel(const __nv_bfloat16* __restrict__ x, int T, int d, int E, const int32_t* __restrict__ ids,
                const int32_t* __restrict__ block_pre, const DevPlan* __restrict__ plan,
                const __grid_constant__ RowTargets targets, uint32_t* __restrict__ row_code,
                const __grid_constant__ PeerSignal sig, int32_t* __restrict__ perm_src,
                int32_t* __restrict__ row_owner, const __grid_constant__ LocalPlan lp) {
  __shared__ uint32_t codes[32 * K];
  // the block's prefix row and the plan tables the ranking reads, staged once
  // (coalesced) so the ranking never waits on L2
  __shared__ int s_pre[kMaxExperts], s_n[kMaxExperts], s_rbase[kMaxExperts + 1];
  __shared__ uint32_t s_mask[kMaxExperts];  // tokens of this block that chose expert e
  __shared__ int s_rrow[kMaxReplicas];
  __shared__ unsigned char s_rrem[kMaxReplicas];
  __shared__ __nv_bfloat16* s_tgt[kMaxTargets];
  griddep_wait();  // launched programmatically behind the block prefix
  const int b = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = lane_id();
  const int t_base = b * 32;
  const int ntok = min(32, T - t_base);
  if (lp.counts) {
    // fused local plan: one merged replica per expert, rows in expert order
    for (int i = threadIdx.x; i < E; i += blockDim.x) {
      int pre = 0;
      for (int bb = 0; bb < b; ++bb) pre += lp.block_counts[(size_t)bb * E + i];
      s_pre[i] = pre;
      s_rbase[i] = i;
      s_rrem[i] = 0;
      s_mask[i] = 0u;
    }
    if (warp == 0) {
      const bool writer = blockIdx.x == 0 && blockIdx.y == 0;
      int row_carry = 0, seg_carry = 0;
      for (int e0 = 0; e0 < E; e0 += 32) {
        const int e = e0 + lane;
        const int n = e < E ? lp.counts[e] : 0;
        int incl = n;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const int v = __shfl_up_sync(0xffffffffu, incl, off);
          if (lane >= off) incl += v;
        }
        const uint32_t active = __ballot_sync(0xffffffffu, n > 0);
        const int row0 = row_carry + incl - n;
        if (e < E) {
          s_n[e] = n;
          s_rrow[e] = row0;
          if (writer) {
            lp.out->n_e[e] = n;
            lp.out->src_off[e] = 0;
            lp.out->rep_base[e] = e;
            lp.out->rep_row_base[e] = row0;
            lp.out->rep_remote[e] = 0;
            if (n > 0) lp.out->segs[seg_carry + __popc(active & ((1u << lane) - 1u))] = GemmSeg{row0, n, e, 0};
          }
        }
        row_carry += __shfl_sync(0xffffffffu, incl, 31);
        seg_carry += __popc(active);
      }
      if (writer && lane == 0) {
        lp.out->E = E;
        lp.out->R = E;
        lp.out->G = 1;
        lp.out->rank = 0;
        lp.out->nseg = seg_carry;
        lp.out->rows_local = row_carry;
        lp.out->rows_send = 0;
        lp.out->rep_base[E] = E;
      }
      // the GEMMs (launched programmatically behind this grid) read the segment
      // list before their griddepcontrol.wait: publish it before this CTA triggers
      if (writer) __threadfence();
    }
    if (threadIdx.x == 0) s_rbase[E] = E;
  } else {
    const int R = plan->R;
    for (int i = threadIdx.x; i < E; i += blockDim.x) {
      s_pre[i] = block_pre[(size_t)b * E + i];
      s_n[i] = plan->n_e[i];
      s_rbase[i] = plan->rep_base[i];
      s_mask[i] = 0u;
    }
    if (threadIdx.x == 0) s_rbase[E] = plan->rep_base[E];
    for (int i = threadIdx.x; i < R; i += blockDim.x) {
      s_rrow[i] = plan->rep_row_base[i];
      s_rrem[i] = static_cast<unsigned char>(plan->rep_remote[i]);
    }
  }
#pragma unroll
  for (int i = 0; i < kMaxTargets; ++i)  // constant indices: the table stays in parameter space
    if (threadIdx.x == i) s_tgt[i] = static_cast<__nv_bfloat16*>(targets.base[i]);
  __syncthreads();

  {
    // stable rank of (token, expert) inside the block = number of EARLIER
    // tokens of the block that chose the same expert: one bit per token.  The
    // K slots are spread over the CTA's warps (slot j on warp j mod kRankWarps):
    // every warp first sets its slots' bits, then ranks them.
    constexpr int kRankWarps = 4;  // blockDim.x / 32
    constexpr int kMine = (K + kRankWarps - 1) / kRankWarps;
    const int t = t_base + lane;
    const bool live = lane < ntok;
    int my[kMine];
#pragma unroll
    for (int q = 0; q < kMine; ++q) {
      const int j = warp + q * kRankWarps;
      my[q] = live && j < K ? ids[(size_t)t * K + j] : -1;
      if (my[q] >= 0) atomicOr(&s_mask[my[q]], 1u << lane);
    }
    __syncthreads();  // every slot's bit is in the masks
    const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
    for (int q = 0; q < kMine; ++q) {
      const int j = warp + q * kRankWarps;
      const int e = my[q];
      if (e < 0) continue;
      const int gr = s_pre[e] + __popc(s_mask[e] & lt);
      // integer replica split: replica r owns floor(n/R) + [r < n mod R] ranks
      const int Re = s_rbase[e + 1] - s_rbase[e];
      int r = 0;
      if (Re > 1) {
        const int n = s_n[e], qq = n / Re, rem = n % Re;
        r = gr < rem * (qq + 1) ? gr / (qq + 1) : rem + (gr - rem * (qq + 1)) / qq;
      }
      const int f = s_rbase[e] + r;
      const uint32_t code =
          static_cast<uint32_t>(s_rrow[f] + gr) | (static_cast<uint32_t>(s_rrem[f]) << kTargetShift);
      codes[lane * K + j] = code;
      if (blockIdx.y == 0) row_code[(size_t)t * K + j] = code;
      if (perm_src) perm_src[code & kRowMask] = t;  // gathered GEMM1: row -> token
      if (row_owner) row_owner[code & kRowMask] = t * K + j;  // fused combine: row -> (token, slot)
    }
  }
  if (perm_src) {  // single GPU, gathered GEMM1: the rows are read from x in place
    griddep_launch_dependents();
    return;
  }
  __syncthreads();

  // stream rows: this CTA covers 16-byte chunks [c_begin, c_end) of every
  // token row of the block (rows split over gridDim.y CTAs for small
  // batches).  (token, chunk) items are spread over all threads and U loads
  // are issued before any store, so the copy pays one memory latency per U
  // items instead of one per token.
  const int chunks_all = d / 8;
  const int per = (chunks_all + gridDim.y - 1) / gridDim.y;
  const int c_begin = blockIdx.y * per, c_end = min(chunks_all, c_begin + per);
  const int nch = max(0, c_end - c_begin);
  const int items = ntok * nch;
  constexpr int U = 4;
  for (int i0 = threadIdx.x; i0 < items; i0 += blockDim.x * U) {
    int4 v[U];
    int tok[U], ch[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int it = i0 + u * blockDim.x;
      tok[u] = it / nch;
      ch[u] = c_begin + (it - tok[u] * nch);
      if (it < items) v[u] = ld_nc_v4(x + (size_t)(t_base + tok[u]) * d + (size_t)ch[u] * 8);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (i0 + u * blockDim.x >= items) break;
#pragma unroll
      for (int j = 0; j < K; ++j) {
        const uint32_t c = codes[tok[u] * K + j];
        // local rows, the NCCL send buffer or a peer's received rows
        st_v4(s_tgt[c >> kTargetShift] + (size_t)(c & kRowMask) * d + (size_t)ch[u] * 8, v[u]);
      }
    }
  }
  griddep_launch_dependents();  // GEMM1 may launch and stream weights while the last CTAs drain
  if (sig.G > 0) {
    // peer memory: every thread's remote stores are performed system-wide
    // before its CTA counts itself done; the last CTA publishes the epoch
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned total = gridDim.x * gridDim.y;
      if (atomicAdd(sig.counter, 1u) == total - 1) {
        *sig.counter = 0u;
        __threadfence_system();
#pragma unroll
        for (int g = 0; g < 8; ++g)
          if (g < sig.G)
            asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(sig.flags[g] + sig.kind * 8 + sig.src),
                         "r"(*sig.epoch)
                         : "memory");
      }
    }
  }
}

// -------------------------------------------------------------- combine
// MOE_FRONT_TRACE: the latest combine CTA end (%globaltimer, atomicMax into trace[14])
__device__ unsigned long long* g_combine_trace = nullptr;
cudaError_t set_combine_trace(unsigned long long* p) { return cudaMemcpyToSymbol(g_combine_trace, &p, sizeof(p)); }

// MOE_FRONT_TRACE=2: a one-thread marker stamped first in the layer's sequence (trace[15])
__global__ void trace_marker_kernel() {
  if (g_combine_trace) {
    unsigned long long v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    g_combine_trace[15] = v;
  }
}
cudaError_t launch_trace_marker(cudaStream_t s) {
  trace_marker_kernel<<<1, 32, 0, s>>>();
  return cudaGetLastError();
}

template <int K>
__global__ void __launch_bounds__(256)
combine_kernel(const __grid_constant__ RowTargets sources, int T, int d, const uint32_t* __restrict__ row_code,
               const float* __restrict__ wts, __nv_bfloat16* __restrict__ y) {
  __shared__ const __nv_bfloat16* s_src[kMaxTargets];
  griddep_wait();  // launched programmatically behind K4
#pragma unroll
  for (int i = 0; i < kMaxTargets; ++i)
    if (threadIdx.x == i) s_src[i] = static_cast<const __nv_bfloat16*>(sources.base[i]);
  __syncthreads();
  const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int lane = lane_id();
  // columns split over gridDim.y (small batches), tokens over warps
  const int chunks_all = d / 8;
  const int per = (chunks_all + gridDim.y - 1) / gridDim.y;
  const int c_begin = blockIdx.y * per, chunks = min(chunks_all, c_begin + per);
  for (int t = warp_global; t < T; t += nwarps) {
    const __nv_bfloat16* src[K];
    float w[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const uint32_t c = row_code[(size_t)t * K + j];
      src[j] = s_src[c >> kTargetShift] + (size_t)(c & kRowMask) * d;  // local, return buffer or a peer's outputs
      w[j] = wts[(size_t)t * K + j];
    }
    __nv_bfloat16* out = y + (size_t)t * d;
    for (int c0 = c_begin + lane; c0 < chunks; c0 += 32) {
      int4 v[K];
#pragma unroll
      for (int j = 0; j < K; ++j) v[j] = ld_nc_v4(src[j] + (size_t)c0 * 8);
      float acc[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = 0.0f;
#pragma unroll
      for (int j = 0; j < K; ++j) {
        const uint32_t* u = reinterpret_cast<const uint32_t*>(&v[j]);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          acc[2 * i] = fmaf(w[j], bf16lo(u[i]), acc[2 * i]);
          acc[2 * i + 1] = fmaf(w[j], bf16hi(u[i]), acc[2 * i + 1]);
        }
      }
      int4 o;
      o.x = pack_bf16(acc[0], acc[1]);
      o.y = pack_bf16(acc[2], acc[3]);
      o.z = pack_bf16(acc[4], acc[5]);
      o.w = pack_bf16(acc[6], acc[7]);
      st_v4(out + (size_t)c0 * 8, o);
    }
  }
  if (g_combine_trace && threadIdx.x == 0) {
    unsigned long long v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    atomicMax(g_combine_trace + 14, v);
  }
}

// ------------------------------------------------------- on-device plan (G = 1)
// Single GPU: every replica is local and co-located replicas of an expert are
// one GEMM segment, so the dispatch plan is an exclusive scan of the gate
// histogram — built on the device, no host round trip.  Row placement is
// identical to the host plan's (expert e's rows start at sum_{e'<e} n_e').
// Runs as the extra CTA of the block-prefix launch (block_prefix_kernel).
__device__ void plan_local_body(const int32_t* __restrict__ counts, int E, DevPlan* __restrict__ plan) {
  __shared__ int base[kMaxExperts + 1];
  __shared__ int seg_idx[kMaxExperts + 1];
  const int tid = threadIdx.x;
  if (tid == 0) {
    int acc = 0, ns = 0;
    for (int e = 0; e < E; ++e) {
      base[e] = acc;
      seg_idx[e] = ns;
      const int n = counts[e];
      acc += n;
      ns += n > 0 ? 1 : 0;
    }
    base[E] = acc;
    seg_idx[E] = ns;
    plan->E = E;
    plan->R = E;
    plan->G = 1;
    plan->rank = 0;
    plan->nseg = ns;
    plan->rows_local = acc;
    plan->rows_send = 0;
    plan->rep_base[E] = E;
  }
  __syncthreads();
  for (int e = tid; e < E; e += blockDim.x) {
    const int n = counts[e];
    plan->n_e[e] = n;
    plan->src_off[e] = 0;
    plan->rep_base[e] = e;  // one (merged) replica per expert
    plan->rep_row_base[e] = base[e];
    plan->rep_remote[e] = 0;
    if (n > 0) plan->segs[seg_idx[e]] = GemmSeg{base[e], n, e, 0};
  }
}


// ---------------------------------------------- on-device exchange plan (G > 1)
// Peer-memory exchange with a placement decided BEFORE the layer (FIXED, or
// MOE_PLAN_PREDICTED planned d layers ahead): every rank derives the same
// direct plan as exchange_plan.cpp (direct mode) from the gathered
// histograms — integer replica split, per-GPU segment layout in replica
// order, this rank's merged segments — without a host round trip.
__global__ void __launch_bounds__(512)
plan_exchange_kernel(const int32_t* __restrict__ counts_all, int stride, int G, int rank,
                     const PlacementTable* __restrict__ pt, DevPlan* __restrict__ plan) {
  __shared__ int s_n[kMaxExperts], s_off[kMaxExperts], s_mine[kMaxExperts];
  __shared__ int s_lrows[kMaxExperts], s_lfirst[kMaxExperts];
  __shared__ int s_start[kMaxReplicas], s_size[kMaxReplicas], s_gpu[kMaxReplicas];
  __shared__ int s_send;
  const int tid = threadIdx.x;
  const int E = pt->E, R = pt->R;
  for (int e = tid; e < E; e += blockDim.x) {
    int n = 0, off = 0;
    for (int g = 0; g < G; ++g) {
      const int c = counts_all[g * stride + e];
      if (g < rank) off += c;
      n += c;
    }
    s_n[e] = n;
    s_off[e] = off;
    s_mine[e] = counts_all[rank * stride + e];
    s_lrows[e] = 0;
    s_lfirst[e] = 0x7fffffff;
    plan->n_e[e] = n;
    plan->src_off[e] = off;
    plan->rep_base[e] = pt->rep_base[e];
  }
  if (tid == 0) {
    plan->rep_base[E] = R;
    s_send = 0;
  }
  __syncthreads();
  for (int f = tid; f < R; f += blockDim.x) {
    const int e = pt->expert_of[f];
    const int rb = pt->rep_base[e], Re = pt->rep_base[e + 1] - rb, r = f - rb;
    const int n = s_n[e], q = n / Re, rem = n % Re;
    s_size[f] = q + (r < rem ? 1 : 0);
    s_start[f] = r * q + min(r, rem);
    s_gpu[f] = pt->gpu_of[f];
  }
  __syncthreads();
  for (int f = tid; f < R; f += blockDim.x) {
    const int g = s_gpu[f], size = s_size[f], start = s_start[f];
    int seg = 0;  // rows of earlier replicas on the same GPU (replica-order layout)
    for (int h = 0; h < f; ++h) seg += s_gpu[h] == g ? s_size[h] : 0;
    plan->rep_row_base[f] = seg - start;
    plan->rep_remote[f] = g;
    const int e = pt->expert_of[f];
    if (g == rank) {
      if (size > 0) {
        atomicAdd(&s_lrows[e], size);
        atomicMin(&s_lfirst[e], seg);
      }
    } else {
      const int lo = max(start, s_off[e]), hi = min(start + size, s_off[e] + s_mine[e]);
      if (hi > lo) atomicAdd(&s_send, hi - lo);
    }
  }
  __syncthreads();
  // this rank's local replicas of one expert are adjacent in its buffer: one
  // GEMM segment per expert with rows here, in expert order
  for (int e = tid; e < E; e += blockDim.x) {
    if (s_lrows[e] == 0) continue;
    int idx = 0;
    for (int h = 0; h < e; ++h) idx += s_lrows[h] > 0 ? 1 : 0;
    plan->segs[idx] = GemmSeg{s_lfirst[e], s_lrows[e], pt->slot_of[e], 0};
  }
  if (tid == 0) {
    int nseg = 0, rows = 0;
    for (int e = 0; e < E; ++e) {
      nseg += s_lrows[e] > 0 ? 1 : 0;
      rows += s_lrows[e];
    }
    plan->E = E;
    plan->R = R;
    plan->G = G;
    plan->rank = rank;
    plan->nseg = nseg;
    plan->rows_local = rows;
    plan->rows_send = s_send;
  }
}

cudaError_t launch_plan_exchange(const int32_t* counts_all, int stride, int G, int rank, const PlacementTable* pt,
                                 DevPlan* plan, cudaStream_t s) {
  plan_exchange_kernel<<<1, 512, 0, s>>>(counts_all, stride, G, rank, pt, plan);
  return cudaGetLastError();
}

// ------------------------------------------------------- small SM copies
// Copies a few KB between device memory and MAPPED pinned host memory with
// the SMs instead of a copy engine, so control data (gate histogram out,
// exchange plan / gate weights in) never queues behind the 100+ MB token
// uploads and result downloads that the pipelined host API keeps in flight.
__global__ void __launch_bounds__(256) small_copy_kernel(int4* __restrict__ dst, const int4* __restrict__ src, int n16) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += gridDim.x * blockDim.x) dst[i] = src[i];
}

// Decode: the first expert weights the swap-AB K4 will stream, pulled into L2
// on a side stream while the gate / dispatch front end runs (they use little
// HBM bandwidth).  One thread per CTA issues bulk prefetches of 256 KB pieces.
__global__ void __launch_bounds__(32) l2_prefetch_kernel(const uint8_t* __restrict__ base, size_t bytes) {
  constexpr size_t kPiece = 256 * 1024;
  if (threadIdx.x != 0) return;
  for (size_t off = static_cast<size_t>(blockIdx.x) * kPiece; off < bytes; off += static_cast<size_t>(gridDim.x) * kPiece) {
    const size_t n = bytes - off < kPiece ? bytes - off : kPiece;
    bulk_prefetch_l2(base + off, static_cast<uint32_t>(n & ~size_t(15)));
  }
}

cudaError_t launch_l2_prefetch(const void* base, size_t bytes, cudaStream_t s) {
  if (!base || bytes < 16) return cudaSuccess;
  l2_prefetch_kernel<<<16, 32, 0, s>>>(static_cast<const uint8_t*>(base), bytes);
  return cudaGetLastError();
}

cudaError_t launch_small_copy(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (bytes == 0) return cudaSuccess;
  if ((bytes & 15) || (reinterpret_cast<uintptr_t>(dst) & 15) || (reinterpret_cast<uintptr_t>(src) & 15))
    return cudaErrorInvalidValue;
  const int n16 = static_cast<int>(bytes / 16);
  const int blocks = n16 / 256 + 1 < 64 ? n16 / 256 + 1 : 64;
  small_copy_kernel<<<blocks, 256, 0, s>>>(static_cast<int4*>(dst), static_cast<const int4*>(src), n16);
  return cudaGetLastError();
}

// ------------------------------------------------------------- launchers
// Programmatic dependent launch: the kernel may be scheduled while its
// predecessor drains and waits in griddepcontrol.wait before touching its
// inputs, which hides the launch gap between the small per-layer kernels.
template <class... KArgs, class... Args>
static cudaError_t launch_pdl(bool pdl, void (*kernel)(KArgs...), dim3 grid, dim3 block, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

cudaError_t launch_block_prefix(const int32_t* block_counts, int nblk, int E, const DevPlan* plan,
                                int32_t* block_pre, cudaStream_t s, const int32_t* local_counts, bool pdl) {
  if (nblk <= 0 && !local_counts) return cudaSuccess;
  // with local_counts: + one CTA that builds the single-GPU plan into *plan
  return launch_pdl(pdl, block_prefix_kernel, dim3(E + (local_counts ? 1 : 0)), dim3(512), s, block_counts, nblk, E, plan,
                    block_pre, local_counts, const_cast<DevPlan*>(plan));
}

#define MOE_SWITCH_K(k, ...)                         \
  switch (k) {                                        \
    case 1: { constexpr int KK = 1; __VA_ARGS__; } break; \
    case 2: { constexpr int KK = 2; __VA_ARGS__; } break; \
    case 4: { constexpr int KK = 4; __VA_ARGS__; } break; \
    case 6: { constexpr int KK = 6; __VA_ARGS__; } break; \
    case 8: { constexpr int KK = 8; __VA_ARGS__; } break; \
    default: return cudaErrorInvalidValue;            \
  }

cudaError_t launch_dispatch(const __nv_bfloat16* x, int T, int d, int E, int k, const int32_t* ids,
                            const int32_t* block_pre, const DevPlan* plan, const RowTargets& targets,
                            uint32_t* row_code, const PeerSignal& sig, cudaStream_t s, int32_t* perm_src,
                            int32_t* row_owner, bool pdl, const int32_t* local_counts,
                            const int32_t* block_counts, DevPlan* plan_out) {
  if (T <= 0) return cudaSuccess;
  if (d % 8) return cudaErrorInvalidValue;
  const int nblk = (T + 31) / 32;
  const LocalPlan lp{local_counts, block_counts, plan_out};
  // at least ~2 CTAs per SM: split each row's chunks when there are few blocks
  // (ranking only when GEMM1 gathers the rows itself)
  const int split = perm_src ? 1 : std::max(1, std::min((2 * 148 + nblk - 1) / nblk, d / 8 / 16));
  const dim3 grid(nblk, split);
  MOE_SWITCH_K(k, return launch_pdl(pdl, dispatch_kernel<KK>, grid, dim3(128), s, x, T, d, E, ids, block_pre, plan,
                                    targets, row_code, sig, perm_src, row_owner, lp));
  return cudaSuccess;
}

bool dispatch_fuses_plan(int T) { return T > 0 && (T + 31) / 32 <= kFusedPlanMaxBlocks; }

cudaError_t launch_combine(const RowTargets& sources, int T, int d, int k, const uint32_t* row_code,
                           const float* wts, __nv_bfloat16* y, int num_sms, cudaStream_t s, bool pdl) {
  if (T <= 0) return cudaSuccess;
  if (d % 8) return cudaErrorInvalidValue;
  const int warps_needed = T;
  int ctas = (warps_needed + 7) / 8;
  ctas = ctas < num_sms * 8 ? ctas : num_sms * 8;
  const int split = std::max(1, std::min((2 * num_sms + ctas - 1) / ctas, d / 8 / 32));
  const dim3 grid(ctas, split);
  MOE_SWITCH_K(k, return launch_pdl(pdl, combine_kernel<KK>, grid, dim3(256), s, sources, T, d, row_code, wts, y));
  return cudaSuccess;
}

// Load every kernel of this file now (CUDA 12 loads kernels lazily on first
// launch, and a lazy load may wait for the whole context — including a
// peer-exchange kernel spinning on another rank that shares the context).
cudaError_t preload_dispatch_kernels() {
  cudaFuncAttributes a;
  const void* fns[] = {
      reinterpret_cast<const void*>(block_prefix_kernel),  reinterpret_cast<const void*>(dispatch_kernel<1>),
      reinterpret_cast<const void*>(l2_prefetch_kernel),
      reinterpret_cast<const void*>(dispatch_kernel<2>),   reinterpret_cast<const void*>(dispatch_kernel<4>),
      reinterpret_cast<const void*>(dispatch_kernel<6>),   reinterpret_cast<const void*>(dispatch_kernel<8>),
      reinterpret_cast<const void*>(combine_kernel<1>),    reinterpret_cast<const void*>(combine_kernel<2>),
      reinterpret_cast<const void*>(combine_kernel<4>),    reinterpret_cast<const void*>(combine_kernel<6>),
      reinterpret_cast<const void*>(combine_kernel<8>),
      reinterpret_cast<const void*>(plan_exchange_kernel), reinterpret_cast<const void*>(small_copy_kernel)};
  for (const void* f : fns) {
    const cudaError_t e = cudaFuncGetAttributes(&a, f);
    if (e != cudaSuccess) return e;
  }
  // The decode weight prefetch runs beside the front end and the swap-AB K4
  // (~200 KB of shared memory per CTA): with the default carveout an SM that
  // hosts a prefetch CTA cannot take a K4 CTA until it drains and reconfigures
  // (K4 CTAs on those SMs started ~8 us late, profiles/ab_frontend_r02.md).
  return cudaFuncSetAttribute(reinterpret_cast<const void*>(l2_prefetch_kernel),
                              cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
}

}  // namespace moe
