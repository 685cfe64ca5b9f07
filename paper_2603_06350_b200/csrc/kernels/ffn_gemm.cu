// ffn_gemm.cu — K4: the expert SwiGLU FFN as two persistent grouped GEMMs on
// 5th-generation tensor cores (tcgen05 + TMEM), fed by TMA over ragged
// per-replica segments.
//
// It is the real work behind the reference's compute term alpha * max_share
// (proj/src/cost_model.cpp:115): each replica segment of the permuted token
// buffer is multiplied by its expert's weights.
//
//   GEMM1 (EPI_SWIGLU): H[r, f] = silu(X[r,:] W1[f,:]) * (X[r,:] W3[f,:])
//       A = X  [rows, d]  K-major;  B = W13 [slot][2ff, d] K-major, W1/W3 rows
//       interleaved in 128-row blocks so one 128x256 accumulator tile holds the
//       gate and up projections of the same 128 ff-columns; the epilogue
//       applies silu(g)*u and writes a 128x128 bf16 tile of H.
//   GEMM2 (EPI_STORE):  Y[r, n] = H[r,:] W2[n,:]
//       A = H  [rows, ff] K-major;  B = W2 [slot][d, ff] K-major.
//
// Kernel anatomy (one CTA per SM, persistent, 6 warps):
//   warp 0      TMA producer: 128x64 A tile + 256x64 B tile per stage (48 KB),
//               4-stage smem ring guarded by full/empty mbarriers.
//   warp 1      TMEM owner + MMA issuer: one elected thread issues
//               tcgen05.mma.cta_group::1.kind::f16 (M=128, N=256, K=16) x4 per
//               stage into a double-buffered TMEM accumulator (2 x 256 cols),
//               tcgen05.commit frees smem stages and publishes finished tiles.
//   warps 2..5  epilogue: tcgen05.ld 32 lanes x 32 cols -> registers ->
//               (silu*mul) -> bf16 -> global; warp w reads TMEM lanes
//               32*(w%4)..+31 as the hardware requires.
// Tile order: segments in (expert, ordinal) order; inside a segment, groups of
// up to 16 m-tiles sweep all n-tiles so concurrently running CTAs share A
// rows and B columns through L2.
#include <atomic>
#include <cstdint>
#include <cuda.h>

#include "dispatch_plan.h"
#include "sm100_ptx.cuh"

namespace moe {

constexpr int kMaxSegs = kMaxReplicas;
constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
// m-tiles swept per n column: GEMM1 (K = d) keeps a whole expert's A rows L2-resident
// while its weights stream once; GEMM2 (K = ff, 3.7 MB A tiles) uses a smaller group.
template <int EPI> constexpr int kGroupM = EPI == 0 ? 32 : 16;
constexpr uint32_t kStageBytesA = BM * BK * 2, kStageBytesB = BN * BK * 2;
constexpr uint32_t kStageBytes = kStageBytesA + kStageBytesB;
constexpr int kThreads = 192;
constexpr uint32_t kTmemCols = 512;

enum : int { EPI_SWIGLU = 0, EPI_STORE = 1 };

// dynamic tile scheduler: the producer warp claims tiles from a global
// counter and hands their ids to the MMA and epilogue warps through a ring
constexpr int kTileRing = 8;

struct SmemLayout {
  // offsets relative to the 1024-aligned base
  static constexpr uint32_t a = 0;
  static constexpr uint32_t b = a + STAGES * kStageBytesA;
  static constexpr uint32_t bars = b + STAGES * kStageBytesB;       // 8-byte mbarriers
  static constexpr uint32_t n_bars = 2 * STAGES + 4 + 2 * kTileRing;
  static constexpr uint32_t tmem_slot = bars + n_bars * 8;
  static constexpr uint32_t tile_ring = tmem_slot + 16;              // int[kTileRing]
  static constexpr uint32_t seg_tiles = tile_ring + kTileRing * 4;   // int[kMaxSegs + 1]
  static constexpr uint32_t segs = seg_tiles + (kMaxSegs + 1) * 4 + 12;  // int4[kMaxSegs]
  static constexpr uint32_t end = ((segs + 15) / 16) * 16 + kMaxSegs * 16;
};
constexpr uint32_t kSmemBytes = SmemLayout::end + 1024;

struct TileCoord {
  int seg, m, n;
};

template <int GM, int TILE_M = BM>
__device__ __forceinline__ TileCoord decode_tile(int t, const int* seg_tiles, const int4* segs, int nseg,
                                                 int n_tiles, int gm_rt = 0) {
  const int GMv = gm_rt > 0 ? gm_rt : GM;
  // binary search: last s with seg_tiles[s] <= t
  int lo = 0, hi = nseg - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (seg_tiles[mid] <= t) lo = mid; else hi = mid - 1;
  }
  const int s = lo;
  const int local = t - seg_tiles[s];
  const int m_tiles = (segs[s].y + TILE_M - 1) / TILE_M;
  const int per_group = GMv * n_tiles;
  const int g = local / per_group;
  const int gm = min(GMv, m_tiles - g * GMv);
  const int rem = local - g * per_group;
  TileCoord c;
  c.seg = s;
  c.n = rem / gm;
  c.m = g * GMv + rem % gm;
  return c;
}

// silu(g) = g * sigmoid(g) with the fast reciprocal: the product is rounded to
// bf16 right after, and the exact IEEE division made the SwiGLU epilogue the
// longest part of a decode tile (cfg5)
__device__ __forceinline__ float silu(float g) { return __fdividef(g, 1.0f + __expf(-g)); }

// Tile order is the same static sequence (decode_tile) either way; with a
// scheduler counter (sched != nullptr: [0] next tile, [1] CTAs done, zero
// before the launch, reset by the last CTA) tiles are CLAIMED in that order by
// whichever CTA's producer is free, so SMs that draw less bandwidth take
// fewer tiles instead of finishing last.
template <int EPI>
__global__ void __launch_bounds__(kThreads, 1)
grouped_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const GemmSeg* __restrict__ segs_g, const int* __restrict__ nseg_g, int n_total,
                    int k_total, int b_rows_per_slot, __nv_bfloat16* __restrict__ out, int out_ld,
                    int* __restrict__ sched, const int32_t* __restrict__ a_gather, int group_m,
                    const __grid_constant__ FusedCombine fc) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SmemLayout::bars);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* tfull = bars + 2 * STAGES;
  uint64_t* tempty = bars + 2 * STAGES + 2;
  uint64_t* ring_full = bars + 2 * STAGES + 4;
  uint64_t* ring_empty = ring_full + kTileRing;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + SmemLayout::tmem_slot);
  volatile int* ring = reinterpret_cast<volatile int*>(smem + SmemLayout::tile_ring);
  int* seg_tiles = reinterpret_cast<int*>(smem + SmemLayout::seg_tiles);
  int4* segs = reinterpret_cast<int4*>(smem + SmemLayout::segs);

  const int warp = threadIdx.x >> 5;
  const int lane = lane_id();
  const int nseg = min(*nseg_g, kMaxSegs);
  const int n_tiles = n_total / BN;

  for (int i = threadIdx.x; i < nseg; i += kThreads) segs[i] = reinterpret_cast<const int4*>(segs_g)[i];
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 4); }
    for (int r = 0; r < kTileRing; ++r) { mbar_init(&ring_full[r], 1); mbar_init(&ring_empty[r], 5); }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int s = 0; s < nseg; ++s) {
      seg_tiles[s] = acc;
      acc += ((segs[s].y + BM - 1) / BM) * n_tiles;
    }
    seg_tiles[nseg] = acc;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int total_tiles = nseg > 0 ? seg_tiles[nseg] : 0;
  const int num_kb = k_total / BK;
  // the next kernel (GEMM2 after GEMM1) may launch now: its CTAs take SMs as
  // this grid's CTAs retire and stream their own weights during our tail
  griddep_launch_dependents();

  if (warp == 0 && a_gather) {
    // ------------------------------------------- producer, gathered A rows
    // GEMM1 straight from the token rows (single GPU): permuted row p of the
    // A operand is token a_gather[p] of x, so the dispatch kernel only ranks
    // and never copies rows.  The whole warp produces: lane i gathers rows
    // 4i .. 4i+3 of every A stage with one TMA gather4; lane 0 also loads B.
    int stage = 0;
    uint32_t phase = 0;
    int rslot = 0;
    uint32_t rphase = 0;
    const uint64_t pol_b = policy_evict_last();
    const int rows_end = nseg > 0 ? segs[nseg - 1].x + segs[nseg - 1].y : 0;
    int t = blockIdx.x;
    bool first = true;
    while (true) {
      if (sched) {
        if (lane == 0) t = atomicAdd(sched, 1);
        t = __shfl_sync(0xffffffffu, t, 0);
      }
      mbar_wait(&ring_empty[rslot], rphase ^ 1);
      if (lane == 0) {
        ring[rslot] = t < total_tiles ? t : -1;
        mbar_arrive(&ring_full[rslot]);
      }
      if (++rslot == kTileRing) { rslot = 0; rphase ^= 1; }
      if (t >= total_tiles) break;
      const TileCoord c = decode_tile<kGroupM<EPI>>(t, seg_tiles, segs, nseg, n_tiles, group_m);
      const int a_row = segs[c.seg].x + c.m * BM;
      const int b_row = segs[c.seg].z * b_rows_per_slot + c.n * BN;
      int kb0 = 0;
      if (first) {
        first = false;
        kb0 = num_kb < STAGES ? num_kb : STAGES;
        if (lane == 0)
          for (int kb = 0; kb < kb0; ++kb) {
            mbar_arrive_expect_tx(&full[kb], kStageBytes);
            tma_load_2d_hint(smem + SmemLayout::b + kb * kStageBytesB, &tmB, &full[kb], kb * BK, b_row, pol_b);
          }
        griddep_wait();  // the row list is the previous kernel's output
      }
      int r[4];
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int p = a_row + 4 * lane + v;
        r[v] = p < rows_end ? a_gather[p] : 0;  // rows past the last segment: any valid row
      }
      __syncwarp();
      for (int kb = 0; kb < kb0; ++kb)
        tma_gather4(smem + SmemLayout::a + kb * kStageBytesA + lane * 4 * BK * 2, &tmA, &full[kb], kb * BK, r[0],
                    r[1], r[2], r[3]);
      if (kb0) {
        stage = kb0 == STAGES ? 0 : kb0;
        phase = kb0 == STAGES ? 1u : 0u;
      }
      for (int kb = kb0; kb < num_kb; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        if (lane == 0) {
          mbar_arrive_expect_tx(&full[stage], kStageBytes);
          tma_load_2d_hint(smem + SmemLayout::b + stage * kStageBytesB, &tmB, &full[stage], kb * BK, b_row, pol_b);
        }
        __syncwarp();
        tma_gather4(smem + SmemLayout::a + stage * kStageBytesA + lane * 4 * BK * 2, &tmA, &full[stage], kb * BK,
                    r[0], r[1], r[2], r[3]);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (!sched) t += gridDim.x;
    }
    if (sched && lane == 0 && atomicAdd(sched + 1, 1) == static_cast<int>(gridDim.x) - 1) {
      sched[0] = 0;
      sched[1] = 0;
    }
  } else if (warp == 0) {
    // ---------------------------------------------------------- producer
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      int rslot = 0;
      uint32_t rphase = 0;
      const uint64_t pol_b = policy_evict_last();
      int t = blockIdx.x;
      bool first = true;
      while (true) {
        if (sched) t = atomicAdd(sched, 1);  // claim the next tile in the static order
        mbar_wait(&ring_empty[rslot], rphase ^ 1);
        ring[rslot] = t < total_tiles ? t : -1;  // -1: no more tiles
        mbar_arrive(&ring_full[rslot]);
        if (++rslot == kTileRing) { rslot = 0; rphase ^= 1; }
        if (t >= total_tiles) break;
        const TileCoord c = decode_tile<kGroupM<EPI>>(t, seg_tiles, segs, nseg, n_tiles, group_m);
        const int a_row = segs[c.seg].x + c.m * BM;
        const int b_row = segs[c.seg].z * b_rows_per_slot + c.n * BN;
        int kb0 = 0;
        if (first) {
          // Launched programmatically behind the kernel that produces A: the
          // weight tiles of the first stages do not depend on it, so stream
          // them while that kernel drains, then wait for it before loading A.
          first = false;
          kb0 = num_kb < STAGES ? num_kb : STAGES;
          for (int kb = 0; kb < kb0; ++kb) {
            mbar_arrive_expect_tx(&full[kb], kStageBytes);  // fresh stages: no empty wait
            tma_load_2d_hint(smem + SmemLayout::b + kb * kStageBytesB, &tmB, &full[kb], kb * BK, b_row, pol_b);
          }
          griddep_wait();
          for (int kb = 0; kb < kb0; ++kb)
            tma_load_2d(smem + SmemLayout::a + kb * kStageBytesA, &tmA, &full[kb], kb * BK, a_row);
          stage = kb0 == STAGES ? 0 : kb0;
          phase = kb0 == STAGES ? 1u : 0u;
        }
        for (int kb = kb0; kb < num_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], kStageBytes);
          tma_load_2d(smem + SmemLayout::a + stage * kStageBytesA, &tmA, &full[stage], kb * BK, a_row);
          tma_load_2d_hint(smem + SmemLayout::b + stage * kStageBytesB, &tmB, &full[stage], kb * BK, b_row,
                           pol_b);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (!sched) t += gridDim.x;
      }
      if (sched && atomicAdd(sched + 1, 1) == static_cast<int>(gridDim.x) - 1) {
        // every CTA has made its last claim: reset for the next launch
        sched[0] = 0;
        sched[1] = 0;
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------- MMA issuer
    if (elect_one()) {
      constexpr uint32_t idesc = umma_idesc_bf16(BM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      const uint32_t a_base = smem_u32(smem + SmemLayout::a);
      const uint32_t b_base = smem_u32(smem + SmemLayout::b);
      int rslot = 0;
      uint32_t rphase = 0;
      while (true) {
        mbar_wait(&ring_full[rslot], rphase);
        const int t = ring[rslot];
        mbar_arrive(&ring_empty[rslot]);
        if (++rslot == kTileRing) { rslot = 0; rphase ^= 1; }
        if (t < 0) break;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t adesc = umma_desc_sw128(a_base + stage * kStageBytesA);
          const uint64_t bdesc = umma_desc_sw128(b_base + stage * kStageBytesB);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            tc_mma_bf16(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb | k) != 0 ? 1u : 0u);
          tc_commit(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        tc_commit(&tfull[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    // --------------------------------------------------------- epilogue
    const int quarter = warp & 3;
    if (EPI == EPI_STORE && fc.row_owner) griddep_wait();  // row_owner / weights come from earlier kernels
    int acc = 0;
    uint32_t acc_phase = 0;
    int rslot = 0;
    uint32_t rphase = 0;
    while (true) {
      mbar_wait(&ring_full[rslot], rphase);
      const int t = ring[rslot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&ring_empty[rslot]);
      if (++rslot == kTileRing) { rslot = 0; rphase ^= 1; }
      if (t < 0) break;
      const TileCoord c = decode_tile<kGroupM<EPI>>(t, seg_tiles, segs, nseg, n_tiles, group_m);
      const int4 sg = segs[c.seg];
      const int row = c.m * BM + quarter * 32 + lane;
      const bool valid = row < sg.y;
      // a 32-row band past the segment's end (most of a decode tile) has
      // nothing to store: skip its TMEM loads and math (warp-uniform)
      const bool band_live = c.m * BM + quarter * 32 < sg.y;
      const size_t grow = static_cast<size_t>(sg.x + row);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + acc * BN;
      if (!band_live) {
      } else if constexpr (EPI == EPI_SWIGLU) {
        __nv_bfloat16* dst = out + grow * out_ld + c.n * (BN / 2);
#pragma unroll 1
        for (int ch = 0; ch < BN / 2 / 32; ++ch) {
          uint32_t g[32], u[32];
          tmem_ld_32x32b_x32(taddr + ch * 32, g);
          tmem_ld_32x32b_x32(taddr + BN / 2 + ch * 32, u);
          tc_wait_ld();
          uint32_t packed[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float h0 = silu(__uint_as_float(g[2 * i])) * __uint_as_float(u[2 * i]);
            const float h1 = silu(__uint_as_float(g[2 * i + 1])) * __uint_as_float(u[2 * i + 1]);
            packed[i] = pack_bf16(h0, h1);
          }
          if (valid) {
            int4* p = reinterpret_cast<int4*>(dst + ch * 32);
#pragma unroll
            for (int v = 0; v < 4; ++v)
              p[v] = make_int4(packed[4 * v], packed[4 * v + 1], packed[4 * v + 2], packed[4 * v + 3]);
          }
        }
      } else {
        __nv_bfloat16* dst = out + grow * out_ld + c.n * BN;
#pragma unroll 1
        for (int ch = 0; ch < BN / 32; ++ch) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(taddr + ch * 32, r);
          tc_wait_ld();
          uint32_t packed[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) packed[i] = pack_bf16(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]));
          if (valid) {
            int4* p = reinterpret_cast<int4*>(dst + ch * 32);
#pragma unroll
            for (int v = 0; v < 4; ++v)
              p[v] = make_int4(packed[4 * v], packed[4 * v + 1], packed[4 * v + 2], packed[4 * v + 3]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);  // the accumulator is free before the combine below
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      if constexpr (EPI == EPI_STORE) {
        if (fc.row_owner && valid) {
          // fused combine: this row's 256 columns are in Yp; the last of the
          // token's k rows to get here sums all k in slot order (as
          // combine_kernel: acc = fma(w_j, y_j, acc) from 0) and writes y
          const int own = fc.row_owner[grow];
          const int tok = own / fc.k;
          int32_t* ctr = fc.counters + (size_t)tok * n_tiles + c.n;
          __threadfence();
          if (atomicAdd(ctr, 1) == fc.k - 1) {
            *ctr = 0;  // ready for the next forward
            __threadfence();
            const __nv_bfloat16* src[8];
            float w[8];
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (j < fc.k) {
                src[j] = out + (size_t)(fc.row_code[(size_t)tok * fc.k + j] & kRowMask) * out_ld + c.n * BN;
                w[j] = fc.wts[(size_t)tok * fc.k + j];
              }
            __nv_bfloat16* yrow = static_cast<__nv_bfloat16*>(fc.y) + (size_t)tok * out_ld + c.n * BN;
#pragma unroll 1
            for (int c8 = 0; c8 < BN / 8; ++c8) {
              float a8[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) a8[i] = 0.0f;
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                if (j >= fc.k) break;
                const int4 v = __ldcg(reinterpret_cast<const int4*>(src[j] + c8 * 8));
                const uint32_t* u = reinterpret_cast<const uint32_t*>(&v);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                  a8[2 * i] = fmaf(w[j], bf16lo(u[i]), a8[2 * i]);
                  a8[2 * i + 1] = fmaf(w[j], bf16hi(u[i]), a8[2 * i + 1]);
                }
              }
              *reinterpret_cast<int4*>(yrow + c8 * 8) =
                  make_int4(pack_bf16(a8[0], a8[1]), pack_bf16(a8[2], a8[3]), pack_bf16(a8[4], a8[5]),
                            pack_bf16(a8[6], a8[7]));
            }
          }
        }
      }
    }
  }
  // a CTA without tiles never waited: completing this grid must still imply
  // that the kernel before it completed (stream order for later kernels)
  griddep_wait();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem_base);
  }
}

// One epilogue warp's 32 rows of a 128x256 accumulator -> bf16 (SwiGLU: the
// 128 gate/up column pairs -> 128 columns of H).
#ifndef MOE_EPI_NOSTORE
#define MOE_EPI_NOSTORE 0  // 1: skip the global stores (A/B of the epilogue's cost only; wrong outputs)
#endif
// Line-coalesced form (stage: this warp's 32 x 144 B shared-memory staging
// rows): per 64 output columns every lane parks its row's 128 bytes in smem,
// then each store instruction writes 4 whole 128-byte row segments (8 lanes x
// 16 B per row) instead of 32 half-sectors of 32 different rows: half the L2
// write transactions, +1-2 % tokens/s at cfg2 (profiles/ab_epi_store_r02.md,
// which also measures what GEMM2's output writes cost the board's clock).
// Row stride 144 B: the row writes and the transposed reads are both
// bank-conflict free per phase.
constexpr uint32_t kStageRow = 144;
constexpr uint32_t kStageWarp = 32 * kStageRow;  // bytes per epilogue warp
#ifndef MOE_EPI_STAGED
#define MOE_EPI_STAGED 1  // 0: direct per-lane row stores (A/B)
#endif

__device__ __forceinline__ void st_shared_v4(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
  asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}
__device__ __forceinline__ int4 ld_shared_v4(uint32_t a) {
  int4 r;
  asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(a) : "memory");
  return r;
}
template <int EPI>
__device__ __forceinline__ void store_accumulator_staged(uint32_t taddr, __nv_bfloat16* __restrict__ out, size_t grow,
                                                         bool valid, int n, int out_ld, uint32_t stage) {
  constexpr int kOutCols = EPI == EPI_SWIGLU ? BN / 2 : BN;
  const int lane = lane_id();
  const size_t grow0 = __shfl_sync(0xffffffffu, grow, 0);  // the warp's rows are grow0 + 0..31
  const uint32_t vmask = __ballot_sync(0xffffffffu, valid);
  __nv_bfloat16* dst0 = out + grow0 * out_ld + n * kOutCols;
  const uint32_t my_row = stage + lane * kStageRow;
  const int jr = lane >> 3, c = lane & 7;  // read side: row 4 i + jr, 16-byte chunk c
#pragma unroll 1
  for (int g = 0; g < kOutCols / 64; ++g) {
    uint32_t packed[32];
    if constexpr (EPI == EPI_SWIGLU) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t gt[32], up[32];
        tmem_ld_32x32b_x32(taddr + (2 * g + h) * 32, gt);
        tmem_ld_32x32b_x32(taddr + BN / 2 + (2 * g + h) * 32, up);
        tc_wait_ld();
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float h0 = silu(__uint_as_float(gt[2 * i])) * __uint_as_float(up[2 * i]);
          const float h1 = silu(__uint_as_float(gt[2 * i + 1])) * __uint_as_float(up[2 * i + 1]);
          packed[16 * h + i] = pack_bf16(h0, h1);
        }
      }
    } else {
      uint32_t r0[32], r1[32];
      tmem_ld_32x32b_x32(taddr + g * 64, r0);
      tmem_ld_32x32b_x32(taddr + g * 64 + 32, r1);
      tc_wait_ld();
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        packed[i] = pack_bf16(__uint_as_float(r0[2 * i]), __uint_as_float(r0[2 * i + 1]));
        packed[16 + i] = pack_bf16(__uint_as_float(r1[2 * i]), __uint_as_float(r1[2 * i + 1]));
      }
    }
#pragma unroll
    for (int v = 0; v < 8; ++v)
      st_shared_v4(my_row + 16 * v, packed[4 * v], packed[4 * v + 1], packed[4 * v + 2], packed[4 * v + 3]);
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int j = 4 * i + jr;
      const int4 w = ld_shared_v4(stage + j * kStageRow + 16 * c);
      if (((vmask >> j) & 1u) && !MOE_EPI_NOSTORE) st_v4(dst0 + static_cast<size_t>(j) * out_ld + g * 64 + c * 8, w);
    }
    __syncwarp();  // the next group overwrites the staging rows
  }
}

// GEMM2 with the combine fused for top-2 on one GPU (FusedY, MOE_FUSED_Y): no
// expert-output rows (yp) are written and no combine kernel runs.  Of a
// token's two rows, the first to reach its (token, n tile) counter parks its
// bf16 output (the value yp would hold) in y[t]; the second waits for it and
// writes fmaf(w1, v1, fmaf(w0, v0, 0)) in slot order — the combine kernel's
// arithmetic on the same bf16 rows, so y is bit-identical to the unfused path
// whichever row arrives first.  GEMM2's written footprint halves
// (profiles/ab_epi_store_r02.md).  Two passes over the tile's columns: first
// arrivals park and publish (+2) without waiting; only then do second
// arrivals wait — every awaited publish comes from an epilogue that waits for
// nothing, so no cycle of waits can form.  The second arrival resets the
// counter for the next forward.
struct FusedY {
  const int32_t* row_owner;  // [rows] t * 2 + slot (dispatch)
  const float* wts;          // [T * 2] routing weights
  __nv_bfloat16* y;          // [T, d]
  int32_t* cnt;              // [T * n_tiles], zero between forwards
  int d, n_tiles;
};
__device__ __forceinline__ int4 ld_cg_v4(const void* p) {
  int4 r;
  asm volatile("ld.global.cg.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p) : "memory");
  return r;
}
__device__ __forceinline__ int ld_acquire_gpu_i32(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void store_fused_y(uint32_t taddr, size_t grow, bool valid, int n, uint32_t stage,
                                              const FusedY& fy) {
  const int lane = lane_id();
  int t = 0, slot = 0;
  float w0 = 0.0f, w1 = 0.0f;
  bool first = false;
  int32_t* cnt = nullptr;
  if (valid) {
    const int own = __ldg(fy.row_owner + grow);
    t = own >> 1;
    slot = own & 1;
    w0 = __ldg(fy.wts + 2 * t);
    w1 = __ldg(fy.wts + 2 * t + 1);
    cnt = fy.cnt + static_cast<size_t>(t) * fy.n_tiles + n;
    first = atomicAdd(cnt, 1) == 0;
  }
  const uint32_t vmask = __ballot_sync(0xffffffffu, valid);
  const uint32_t fmask = __ballot_sync(0xffffffffu, first);
  const uint32_t my_row = stage + lane * kStageRow;
  const int jr = lane >> 3, c = lane & 7;
#pragma unroll 1
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 1) {
      // publish the first arrivals (all lanes' stores before the owners' release), then wait
      __threadfence();
      __syncwarp();
      if (valid && first) asm volatile("red.release.gpu.global.add.s32 [%0], 2;" ::"l"(cnt) : "memory");
      if (valid && !first) {
        // bounded: a counter left non-zero by an aborted forward must fail loudly, not hang
        unsigned long long t0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        while (ld_acquire_gpu_i32(cnt) < 4) {
          __nanosleep(64);
          unsigned long long t1;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
          if (t1 - t0 > 2000000000ull) __trap();
        }
      }
      __syncwarp();
    }
    const uint32_t mine = pass == 0 ? (vmask & fmask) : (vmask & ~fmask);
    if (mine == 0u) continue;
#pragma unroll 1
    for (int g = 0; g < BN / 64; ++g) {
      uint32_t r0[32], r1[32];
      tmem_ld_32x32b_x32(taddr + g * 64, r0);
      tmem_ld_32x32b_x32(taddr + g * 64 + 32, r1);
      tc_wait_ld();
      uint32_t packed[32];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        packed[i] = pack_bf16(__uint_as_float(r0[2 * i]), __uint_as_float(r0[2 * i + 1]));
        packed[16 + i] = pack_bf16(__uint_as_float(r1[2 * i]), __uint_as_float(r1[2 * i + 1]));
      }
#pragma unroll
      for (int v = 0; v < 8; ++v)
        st_shared_v4(my_row + 16 * v, packed[4 * v], packed[4 * v + 1], packed[4 * v + 2], packed[4 * v + 3]);
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int j = 4 * i + jr;
        const int tj = __shfl_sync(0xffffffffu, t, j);
        const int sj = __shfl_sync(0xffffffffu, slot, j);
        const float a0 = __shfl_sync(0xffffffffu, w0, j), a1 = __shfl_sync(0xffffffffu, w1, j);
        if ((mine >> j) & 1u) {
          int4 v4 = ld_shared_v4(stage + j * kStageRow + 16 * c);
          __nv_bfloat16* dst = fy.y + static_cast<size_t>(tj) * fy.d + n * BN + g * 64 + c * 8;
          if (pass == 1) {  // slot order: the parked row is the other slot's
            const int4 o = ld_cg_v4(dst);
            const uint32_t own4[4] = {static_cast<uint32_t>(v4.x), static_cast<uint32_t>(v4.y),
                                      static_cast<uint32_t>(v4.z), static_cast<uint32_t>(v4.w)};
            const uint32_t park4[4] = {static_cast<uint32_t>(o.x), static_cast<uint32_t>(o.y),
                                       static_cast<uint32_t>(o.z), static_cast<uint32_t>(o.w)};
            uint32_t res[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const uint32_t s0 = sj == 0 ? own4[q] : park4[q], s1 = sj == 0 ? park4[q] : own4[q];
              const float lo = fmaf(a1, bf16lo(s1), fmaf(a0, bf16lo(s0), 0.0f));
              const float hi = fmaf(a1, bf16hi(s1), fmaf(a0, bf16hi(s0), 0.0f));
              res[q] = pack_bf16(lo, hi);
            }
            v4 = make_int4(static_cast<int>(res[0]), static_cast<int>(res[1]), static_cast<int>(res[2]),
                           static_cast<int>(res[3]));
          }
          st_v4(dst, v4);
        }
      }
      __syncwarp();
    }
  }
  __syncwarp();
  if (valid && !first) *cnt = 0;  // the pair is closed: ready for the next forward
}

template <int EPI>
__device__ __forceinline__ void store_accumulator(uint32_t taddr, __nv_bfloat16* __restrict__ out, size_t grow,
                                                  bool valid, int n, int out_ld) {
  if constexpr (EPI == EPI_SWIGLU) {
    __nv_bfloat16* dst = out + grow * out_ld + n * (BN / 2);
#pragma unroll 1
    for (int ch = 0; ch < BN / 2 / 32; ++ch) {
      uint32_t g[32], u[32];
      tmem_ld_32x32b_x32(taddr + ch * 32, g);
      tmem_ld_32x32b_x32(taddr + BN / 2 + ch * 32, u);
      tc_wait_ld();
      uint32_t packed[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float h0 = silu(__uint_as_float(g[2 * i])) * __uint_as_float(u[2 * i]);
        const float h1 = silu(__uint_as_float(g[2 * i + 1])) * __uint_as_float(u[2 * i + 1]);
        packed[i] = pack_bf16(h0, h1);
      }
      if (valid && !MOE_EPI_NOSTORE) {
        int4* p = reinterpret_cast<int4*>(dst + ch * 32);
#pragma unroll
        for (int v = 0; v < 4; ++v) p[v] = make_int4(packed[4 * v], packed[4 * v + 1], packed[4 * v + 2], packed[4 * v + 3]);
      }
    }
  } else {
    __nv_bfloat16* dst = out + grow * out_ld + n * BN;
#pragma unroll 1
    for (int ch = 0; ch < BN / 32; ++ch) {
      uint32_t r[32];
      tmem_ld_32x32b_x32(taddr + ch * 32, r);
      tc_wait_ld();
      uint32_t packed[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) packed[i] = pack_bf16(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]));
      if (valid && !MOE_EPI_NOSTORE) {
        int4* p = reinterpret_cast<int4*>(dst + ch * 32);
#pragma unroll
        for (int v = 0; v < 4; ++v) p[v] = make_int4(packed[4 * v], packed[4 * v + 1], packed[4 * v + 2], packed[4 * v + 3]);
      }
    }
  }
}

// ===================================================================
// Cluster-multicast variant ("mc"): a cluster of 2 CTAs computes the two
// vertically adjacent 128x256 tiles m = 2p, 2p+1 of one segment and n tile
// with the 1-SM MMA (cta_group::1, M=128, N=256, own TMEM accumulators).  The
// B tile both need is read from L2 ONCE: each CTA's TMA fetches one 128-row
// half and multicasts it into both CTAs' shared memory, so per SM and k-block
// 16 KB of A + 16 KB of B cross L2 -> SM instead of 48 KB, while every MMA
// operand stays in the CTA's own smem (the cta_group::2 kernel instead reads
// half of B from the peer SM on every MMA).  A stage is free once BOTH CTAs'
// MMAs have read it: each MMA commit arrives multicast on the empty barriers
// of the two CTAs (count 2).  When a segment has an odd number of m-tiles the
// last pair's second CTA has no rows: it loads and multicasts its half of B,
// skips A and the MMAs, and releases each stage with plain cluster arrives.
template <int EPI> constexpr int kGroupMmc = EPI == 0 ? 16 : 8;  // in 256-row pairs

template <int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
grouped_gemm_mc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmBh,
                       const GemmSeg* __restrict__ segs_g, const int* __restrict__ nseg_g, int n_total, int k_total,
                       int b_rows_per_slot, __nv_bfloat16* __restrict__ out, int out_ld, int group_m) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SmemLayout::bars);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* tfull = bars + 2 * STAGES;
  uint64_t* tempty = bars + 2 * STAGES + 2;
  uint64_t* ring_full = bars + 2 * STAGES + 4;
  uint64_t* ring_empty = ring_full + kTileRing;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + SmemLayout::tmem_slot);
  volatile int* ring = reinterpret_cast<volatile int*>(smem + SmemLayout::tile_ring);
  int* seg_tiles = reinterpret_cast<int*>(smem + SmemLayout::seg_tiles);
  int4* segs = reinterpret_cast<int4*>(smem + SmemLayout::segs);

  const int warp = threadIdx.x >> 5;
  const int lane = lane_id();
  const int rank = static_cast<int>(cluster_ctarank());
  const int cluster = blockIdx.x >> 1, num_clusters = gridDim.x >> 1;
  const int nseg = min(*nseg_g, kMaxSegs);
  const int n_tiles = n_total / BN;

  for (int i = threadIdx.x; i < nseg; i += kThreads) segs[i] = reinterpret_cast<const int4*>(segs_g)[i];
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmBh);
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 2); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 4); }
    for (int r = 0; r < kTileRing; ++r) { mbar_init(&ring_full[r], 1); mbar_init(&ring_empty[r], 5); }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int s = 0; s < nseg; ++s) {
      seg_tiles[s] = acc;
      acc += ((segs[s].y + 2 * BM - 1) / (2 * BM)) * n_tiles;
    }
    seg_tiles[nseg] = acc;
  }
  tc_fence_before();
  cluster_sync();  // both CTAs' barriers exist before any multicast or remote arrive
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int total_tiles = nseg > 0 ? seg_tiles[nseg] : 0;
  const int num_kb = k_total / BK;
  griddep_launch_dependents();

  // this CTA's m-tile of pair tile t, and whether it has any rows
  auto my_tile = [&](int t, TileCoord& c) {
    c = decode_tile<kGroupMmc<EPI>, 2 * BM>(t, seg_tiles, segs, nseg, n_tiles, group_m);
    c.m = 2 * c.m + rank;
    return c.m * BM < segs[c.seg].y;
  };

  if (warp == 0) {
    // ---------------------------------------------------------- producer
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      int rslot = 0;
      uint32_t rphase = 0;
      const uint64_t pol_b = policy_evict_last();
      bool first = true;
      for (int t = cluster;; t += num_clusters) {
        mbar_wait(&ring_empty[rslot], rphase ^ 1);
        ring[rslot] = t < total_tiles ? t : -1;
        mbar_arrive(&ring_full[rslot]);
        if (++rslot == kTileRing) { rslot = 0; rphase ^= 1; }
        if (t >= total_tiles) break;
        TileCoord c;
        const bool mine = my_tile(t, c);
        const int a_row = segs[c.seg].x + c.m * BM;
        const int b_row = segs[c.seg].z * b_rows_per_slot + c.n * BN + rank * (BN / 2);
        const uint32_t bytes = (mine ? kStageBytesA : 0u) + kStageBytesB;
        const uint32_t b_off = static_cast<uint32_t>(rank) * (kStageBytesB / 2);
        int kb0 = 0;
        if (first) {
          // weights first (they do not depend on the previous kernel), then A
          first = false;
          kb0 = num_kb < STAGES ? num_kb : STAGES;
          for (int kb = 0; kb < kb0; ++kb) {
            mbar_arrive_expect_tx(&full[kb], bytes);
            tma_load_2d_mc(smem + SmemLayout::b + kb * kStageBytesB + b_off, &tmBh, &full[kb], kb * BK, b_row, 0x3,
                           pol_b);
          }
          griddep_wait();
          if (mine)
            for (int kb = 0; kb < kb0; ++kb)
              tma_load_2d(smem + SmemLayout::a + kb * kStageBytesA, &tmA, &full[kb], kb * BK, a_row);
          stage = kb0 == STAGES ? 0 : kb0;
          phase = kb0 == STAGES ? 1u : 0u;
        }
        for (int kb = kb0; kb < num_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);  // both CTAs have consumed this stage
          mbar_arrive_expect_tx(&full[stage], bytes);
          if (mine) tma_load_2d(smem + SmemLayout::a + stage * kStageBytesA, &tmA, &full[stage], kb * BK, a_row);
          tma_load_2d_mc(smem + SmemLayout::b + stage * kStageBytesB + b_off, &tmBh, &full[stage], kb * BK, b_row,
                         0x3, pol_b);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------- MMA issuer
    if (elect_one()) {
      constexpr uint32_t idesc = umma_idesc_bf16(BM, BN);
      const uint32_t peer_empty0 = mapa_shared(smem_u32(&empty[0]), static_cast<uint32_t>(rank ^ 1));
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      const uint32_t a_base = smem_u32(smem + SmemLayout::a);
      const uint32_t b_base = smem_u32(smem + SmemLayout::b);
      int rslot = 0;
      uint32_t rphase = 0;
      while (true) {
        mbar_wait(&ring_full[rslot], rphase);
        const int t = ring[rslot];
        mbar_arrive(&ring_empty[rslot]);
        if (++rslot == kTileRing) { rslot = 0; rphase ^= 1; }
        if (t < 0) break;
        TileCoord c;
        if (!my_tile(t, c)) {
          // no rows here: release each stage of the shared B on both CTAs
          for (int kb = 0; kb < num_kb; ++kb) {
            mbar_wait(&full[stage], phase);
            mbar_arrive(&empty[stage]);
            mbar_arrive_cluster(peer_empty0 + stage * 8);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
          continue;
        }
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t adesc = umma_desc_sw128(a_base + stage * kStageBytesA);
          const uint64_t bdesc = umma_desc_sw128(b_base + stage * kStageBytesB);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            tc_mma_bf16(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb | k) != 0 ? 1u : 0u);
          tc_commit_mc(&empty[stage], 0x3);  // this CTA has read the stage: tell both producers
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        tc_commit(&tfull[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    // --------------------------------------------------------- epilogue
    const int quarter = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    int rslot = 0;
    uint32_t rphase = 0;
    while (true) {
      mbar_wait(&ring_full[rslot], rphase);
      const int t = ring[rslot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&ring_empty[rslot]);
      if (++rslot == kTileRing) { rslot = 0; rphase ^= 1; }
      if (t < 0) break;
      TileCoord c;
      if (!my_tile(t, c)) continue;
      const int4 sg = segs[c.seg];
      const int row = c.m * BM + quarter * 32 + lane;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      if (c.m * BM + quarter * 32 < sg.y) {
        const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + acc * BN;
        store_accumulator<EPI>(taddr, out, static_cast<size_t>(sg.x + row), row < sg.y, c.n, out_ld);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }
  griddep_wait();
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // the peer must not exit while this CTA still multicasts into it
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem_base);
  }
}

// ===================================================================
// 2-CTA variant: a cluster of 2 SMs computes a 256x256 tile with
// tcgen05.mma.cta_group::2 (M=256).  Each CTA stages its own 128 A rows and
// HALF of the 256 B rows (the W1 block on CTA 0, the W3 block on CTA 1 for
// GEMM1), so per SM and k-block it moves 32 KB instead of 48 KB through
// L2 -> smem for the same MMA work; both CTAs' TMA bytes land on the leader's
// full barrier, the leader's single MMA thread issues for the pair, commits
// multicast to both CTAs' empty / tmem-full barriers, and both CTAs' epilogue
// warps (each reading its own TMEM: 128 rows x 256 cols) release the
// accumulator on the leader's tmem-empty barrier (8 arrivals).  Tiles reach
// both CTAs through a ring the leader's producer fills: statically (cluster c
// takes c, c + clusters, ...) or, with a scheduler counter (MOE_GEMM_SCHED=
// dynamic), claimed in tile order so the clusters in flight always cover one
// contiguous window of tiles; every consumer of both CTAs frees a slot on the
// leader's ring-empty barrier (10 arrivals).
constexpr int BM2 = 256;                 // rows per cluster tile
constexpr int STAGES2 = 6;
constexpr uint32_t kHalfA = 128 * BK * 2, kHalfB = 128 * BK * 2;  // 16 KB each, per CTA
constexpr uint32_t kStage2 = kHalfA + kHalfB;

template <int EPI> constexpr int kGroupM2 = EPI == 0 ? 16 : 8;  // in 256-row tiles

struct SmemLayout2 {
  static constexpr uint32_t a = 0;
  static constexpr uint32_t b = a + STAGES2 * kHalfA;
  static constexpr uint32_t bars = b + STAGES2 * kHalfB;
  static constexpr uint32_t n_bars = 2 * STAGES2 + 4 + 2 * kTileRing;
  static constexpr uint32_t tmem_slot = bars + n_bars * 8;
  static constexpr uint32_t tile_ring = tmem_slot + 16;              // int[kTileRing]
  static constexpr uint32_t seg_tiles = tile_ring + kTileRing * 4;
  static constexpr uint32_t segs = seg_tiles + (kMaxSegs + 1) * 4 + 12;
  static constexpr uint32_t epi_stage = ((segs + 15) / 16) * 16 + kMaxSegs * 16;  // 4 epilogue warps
  static constexpr uint32_t end = epi_stage + 4 * kStageWarp;
};
constexpr uint32_t kSmemBytes2 = SmemLayout2::end + 1024;
static_assert(kSmemBytes2 <= 232448, "smem budget (2-CTA)");

template <int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
grouped_gemm_2sm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        const GemmSeg* __restrict__ segs_g, const int* __restrict__ nseg_g, int n_total, int k_total,
                        int b_rows_per_slot, __nv_bfloat16* __restrict__ out, int out_ld, int group_m, int l2pol,
                        int* __restrict__ sched, const __grid_constant__ FusedY fy) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SmemLayout2::bars);
  uint64_t* full = bars;                      // used on the leader only
  uint64_t* empty = bars + STAGES2;           // per CTA
  uint64_t* tfull = bars + 2 * STAGES2;       // per CTA
  uint64_t* tempty = bars + 2 * STAGES2 + 2;  // used on the leader only (8 arrivals)
  uint64_t* ring_full = bars + 2 * STAGES2 + 4;      // per CTA (1 arrival: the leader's producer)
  uint64_t* ring_empty = ring_full + kTileRing;      // used on the leader only (10 arrivals)
  volatile int* ring = reinterpret_cast<volatile int*>(smem + SmemLayout2::tile_ring);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + SmemLayout2::tmem_slot);
  int* seg_tiles = reinterpret_cast<int*>(smem + SmemLayout2::seg_tiles);
  int4* segs = reinterpret_cast<int4*>(smem + SmemLayout2::segs);

  const int warp = threadIdx.x >> 5;
  const int lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cluster = blockIdx.x >> 1, num_clusters = gridDim.x >> 1;
  const int nseg = min(*nseg_g, kMaxSegs);
  const int n_tiles = n_total / BN;

  for (int i = threadIdx.x; i < nseg; i += kThreads) segs[i] = reinterpret_cast<const int4*>(segs_g)[i];
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES2; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 8); }
    for (int r = 0; r < kTileRing; ++r) { mbar_init(&ring_full[r], 1); mbar_init(&ring_empty[r], 10); }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_2sm<kTmemCols>(tmem_slot);
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int s = 0; s < nseg; ++s) {
      seg_tiles[s] = acc;
      acc += ((segs[s].y + BM2 - 1) / BM2) * n_tiles;
    }
    seg_tiles[nseg] = acc;
  }
  tc_fence_before();
  cluster_sync();  // barriers of both CTAs initialised before any remote arrive / TMA
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int total_tiles = nseg > 0 ? seg_tiles[nseg] : 0;
  const int num_kb = k_total / BK;
  // the next kernel (GEMM2 after GEMM1) may launch now and stream its weights
  // while this grid's CTAs retire
  griddep_launch_dependents();

  if (warp == 0) {
    // ---------------------------------------------------------- producer (both CTAs)
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      // A tiles are reused by every n tile of the group: evict_first here made
      // GEMM1 re-read them from HBM (21 GB per launch instead of 3 GB)
      // l2pol (MOE_GEMM_L2POL, A/B): bits 0-1 A, bits 2-3 B: 0 evict_normal,
      // 1 evict_last, 2 evict_first; default A normal, B evict_last
      auto pol = [](int v) {
        return v == 1 ? policy_evict_last() : v == 2 ? policy_evict_first() : policy_evict_normal();
      };
      const uint64_t pol_a = pol(l2pol & 3), pol_b = pol((l2pol >> 2) & 3);
      const uint32_t peer_ring = mapa_shared(smem_u32(const_cast<int*>(ring)), 1);
      const uint32_t peer_ring_full0 = mapa_shared(smem_u32(&ring_full[0]), 1);
      const uint32_t leader_ring_empty0 = mapa_shared(smem_u32(&ring_empty[0]), 0);
      int rslot = 0;
      uint32_t rphase = 0;
      bool first = true;
      for (int k_static = 0;; ++k_static) {
        int t;
        if (leader) {  // claim the next tile and hand it to both CTAs
          mbar_wait(&ring_empty[rslot], rphase ^ 1);
          t = sched ? atomicAdd(sched, 1) : cluster + k_static * num_clusters;
          if (t >= total_tiles) t = -1;
          ring[rslot] = t;
          st_shared_cluster(peer_ring + rslot * 4, t);
          mbar_arrive(&ring_full[rslot]);
          mbar_arrive_cluster(peer_ring_full0 + rslot * 8);  // release: the store above is visible first
        } else {
          mbar_wait(&ring_full[rslot], rphase);
          t = ring[rslot];
          mbar_arrive_cluster(leader_ring_empty0 + rslot * 8);
        }
        if (++rslot == kTileRing) { rslot = 0; rphase ^= 1; }
        if (t < 0) break;
        const TileCoord c = decode_tile<kGroupM2<EPI>, BM2>(t, seg_tiles, segs, nseg, n_tiles, group_m);
        const int a_row = segs[c.seg].x + c.m * BM2 + static_cast<int>(rank) * 128;
        const int b_row = segs[c.seg].z * b_rows_per_slot + c.n * BN + static_cast<int>(rank) * 128;
        int kb0 = 0;
        if (first) {
          // launched programmatically behind the kernel that produces A: stream
          // the first weight stages while it drains, then wait for it
          first = false;
          kb0 = num_kb < STAGES2 ? num_kb : STAGES2;
          for (int kb = 0; kb < kb0; ++kb) {
            if (leader) mbar_arrive_expect_tx(&full[kb], 2 * kStage2);  // fresh stages: no empty wait
            tma_load_2d_2sm(smem + SmemLayout2::b + kb * kHalfB, &tmB, &full[kb], kb * BK, b_row, pol_b);
          }
          griddep_wait();
          for (int kb = 0; kb < kb0; ++kb)
            tma_load_2d_2sm(smem + SmemLayout2::a + kb * kHalfA, &tmA, &full[kb], kb * BK, a_row, pol_a);
          stage = kb0 == STAGES2 ? 0 : kb0;
          phase = kb0 == STAGES2 ? 1u : 0u;
        }
        for (int kb = kb0; kb < num_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (leader) mbar_arrive_expect_tx(&full[stage], 2 * kStage2);
          tma_load_2d_2sm(smem + SmemLayout2::a + stage * kHalfA, &tmA, &full[stage], kb * BK, a_row, pol_a);
          tma_load_2d_2sm(smem + SmemLayout2::b + stage * kHalfB, &tmB, &full[stage], kb * BK, b_row, pol_b);
          if (++stage == STAGES2) { stage = 0; phase ^= 1; }
        }
      }
      if (leader && sched && atomicAdd(sched + 1, 1) == num_clusters - 1) {
        sched[0] = 0;  // every cluster has made its last claim: reset for the next launch
        sched[1] = 0;
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------- MMA issuer (leader)
    if (leader && elect_one()) {
      constexpr uint32_t idesc = umma_idesc_bf16(BM2, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      const uint32_t a_base = smem_u32(smem + SmemLayout2::a);
      const uint32_t b_base = smem_u32(smem + SmemLayout2::b);
      int rslot = 0;
      uint32_t rphase = 0;
      while (true) {
        mbar_wait(&ring_full[rslot], rphase);
        const int t = ring[rslot];
        mbar_arrive(&ring_empty[rslot]);
        if (++rslot == kTileRing) { rslot = 0; rphase ^= 1; }
        if (t < 0) break;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t adesc = umma_desc_sw128(a_base + stage * kHalfA);
          const uint64_t bdesc = umma_desc_sw128(b_base + stage * kHalfB);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            tc_mma_bf16_2sm(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb | k) != 0 ? 1u : 0u);
          tc_commit_2sm_mc(&empty[stage], 0x3);
          if (++stage == STAGES2) { stage = 0; phase ^= 1; }
        }
        tc_commit_2sm_mc(&tfull[acc], 0x3);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    // --------------------------------------------------------- epilogue (both CTAs)
    const int quarter = warp & 3;
    const uint32_t tempty_leader0 = mapa_shared(smem_u32(&tempty[0]), 0);
    const uint32_t leader_ring_empty0 = mapa_shared(smem_u32(&ring_empty[0]), 0);
    int acc = 0;
    uint32_t acc_phase = 0;
    int rslot = 0;
    uint32_t rphase = 0;
    while (true) {
      mbar_wait(&ring_full[rslot], rphase);
      const int t = ring[rslot];
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(leader_ring_empty0 + rslot * 8);
      if (++rslot == kTileRing) { rslot = 0; rphase ^= 1; }
      if (t < 0) break;
      const TileCoord c = decode_tile<kGroupM2<EPI>, BM2>(t, seg_tiles, segs, nseg, n_tiles, group_m);
      const int4 sg = segs[c.seg];
      const int row = c.m * BM2 + static_cast<int>(rank) * 128 + quarter * 32 + lane;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + acc * BN;
      if (EPI == EPI_STORE && fy.y)
        store_fused_y(taddr, static_cast<size_t>(sg.x + row), row < sg.y, c.n,
                      smem_u32(smem + SmemLayout2::epi_stage) + (warp - 2) * kStageWarp, fy);
      else if (MOE_EPI_STAGED)
        store_accumulator_staged<EPI>(taddr, out, static_cast<size_t>(sg.x + row), row < sg.y, c.n, out_ld,
                                      smem_u32(smem + SmemLayout2::epi_stage) + (warp - 2) * kStageWarp);
      else
        store_accumulator<EPI>(taddr, out, static_cast<size_t>(sg.x + row), row < sg.y, c.n, out_ld);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_leader0 + acc * 8);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }
  griddep_wait();  // a CTA without tiles never waited: keep stream order for later kernels
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // the peer must not exit while the leader still multicasts to it
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_2sm<kTmemCols>(tmem_base);
  }
}

// ===================================================================
// Single-CTA 256-row variant: per k-block the CTA stages a 256x64 A tile and
// a 256x64 B tile (64 KB, 3 stages) and issues two M=128 MMAs (top and
// bottom row halves) that share the B operand, accumulating into the two
// halves of TMEM (2 x 256 columns, single-buffered).  Per FLOP it moves 1/3
// less data from L2 than the 128-row kernel and keeps more bytes in flight
// per MMA cycle, with no cross-SM operand traffic; the price is that the
// epilogue of tile i is not overlapped with the MMAs of tile i+1.
constexpr int BM4 = 256, STAGES4 = 3;
constexpr uint32_t kStageA4 = BM4 * BK * 2, kStageB4 = BN * BK * 2, kStage4 = kStageA4 + kStageB4;

struct SmemLayout4 {
  static constexpr uint32_t a = 0;
  static constexpr uint32_t b = a + STAGES4 * kStageA4;
  static constexpr uint32_t bars = b + STAGES4 * kStageB4;
  static constexpr uint32_t n_bars = 2 * STAGES4 + 2;
  static constexpr uint32_t tmem_slot = bars + n_bars * 8;
  static constexpr uint32_t seg_tiles = tmem_slot + 16;
  static constexpr uint32_t segs = seg_tiles + (kMaxSegs + 1) * 4 + 12;
  static constexpr uint32_t end = ((segs + 15) / 16) * 16 + kMaxSegs * 16;
};
constexpr uint32_t kSmemBytes4 = SmemLayout4::end + 1024;
static_assert(kSmemBytes4 <= 232448, "smem budget (256-row variant)");

template <int EPI>
__global__ void __launch_bounds__(kThreads, 1)
grouped_gemm_m256_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                         const GemmSeg* __restrict__ segs_g, const int* __restrict__ nseg_g, int n_total, int k_total,
                         int b_rows_per_slot, __nv_bfloat16* __restrict__ out, int out_ld) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SmemLayout4::bars);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES4;
  uint64_t* tfull = bars + 2 * STAGES4;
  uint64_t* tempty = bars + 2 * STAGES4 + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + SmemLayout4::tmem_slot);
  int* seg_tiles = reinterpret_cast<int*>(smem + SmemLayout4::seg_tiles);
  int4* segs = reinterpret_cast<int4*>(smem + SmemLayout4::segs);

  const int warp = threadIdx.x >> 5;
  const int lane = lane_id();
  const int nseg = min(*nseg_g, kMaxSegs);
  const int n_tiles = n_total / BN;

  for (int i = threadIdx.x; i < nseg; i += kThreads) segs[i] = reinterpret_cast<const int4*>(segs_g)[i];
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES4; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(tfull, 1);
    mbar_init(tempty, 4);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int s = 0; s < nseg; ++s) {
      seg_tiles[s] = acc;
      acc += ((segs[s].y + BM4 - 1) / BM4) * n_tiles;
    }
    seg_tiles[nseg] = acc;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int total_tiles = nseg > 0 ? seg_tiles[nseg] : 0;
  const int num_kb = k_total / BK;
  constexpr int GM4 = EPI == EPI_SWIGLU ? 16 : 8;  // 256-row tiles per n sweep

  if (warp == 0) {
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      const uint64_t pol_b = policy_evict_last();
      for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
        const TileCoord c = decode_tile<GM4, BM4>(t, seg_tiles, segs, nseg, n_tiles);
        const int a_row = segs[c.seg].x + c.m * BM4;
        const int b_row = segs[c.seg].z * b_rows_per_slot + c.n * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], kStage4);
          tma_load_2d(smem + SmemLayout4::a + stage * kStageA4, &tmA, &full[stage], kb * BK, a_row);
          tma_load_2d_hint(smem + SmemLayout4::b + stage * kStageB4, &tmB, &full[stage], kb * BK, b_row, pol_b);
          if (++stage == STAGES4) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      constexpr uint32_t idesc = umma_idesc_bf16(BM, BN);
      int stage = 0;
      uint32_t phase = 0, acc_phase = 0;
      const uint32_t a_base = smem_u32(smem + SmemLayout4::a);
      const uint32_t b_base = smem_u32(smem + SmemLayout4::b);
      for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
        mbar_wait(tempty, acc_phase ^ 1);
        tc_fence_after();
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_st = a_base + stage * kStageA4;
          const uint64_t a_top = umma_desc_sw128(a_st);
          const uint64_t a_bot = umma_desc_sw128(a_st + BM * 128);  // rows 128..255: +16 KB
          const uint64_t bdesc = umma_desc_sw128(b_base + stage * kStageB4);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint32_t acc = (kb | k) != 0 ? 1u : 0u;
            tc_mma_bf16(tmem_base, a_top + 2 * k, bdesc + 2 * k, idesc, acc);
            tc_mma_bf16(tmem_base + BN, a_bot + 2 * k, bdesc + 2 * k, idesc, acc);
          }
          tc_commit(&empty[stage]);
          if (++stage == STAGES4) { stage = 0; phase ^= 1; }
        }
        tc_commit(tfull);
        acc_phase ^= 1;
      }
    }
  } else {
    const int quarter = warp & 3;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
      const TileCoord c = decode_tile<GM4, BM4>(t, seg_tiles, segs, nseg, n_tiles);
      const int4 sg = segs[c.seg];
      mbar_wait(tfull, acc_phase);
      tc_fence_after();
#pragma unroll 1
      for (int half = 0; half < 2; ++half) {
        const int row = c.m * BM4 + half * BM + quarter * 32 + lane;
        const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + half * BN;
        store_accumulator<EPI>(taddr, out, static_cast<size_t>(sg.x + row), row < sg.y, c.n, out_ld);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty);
      acc_phase ^= 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem_base);
  }
}

cudaError_t launch_grouped_gemm_m256(int epi, const CUtensorMap* tmA, const CUtensorMap* tmB, const GemmSeg* segs,
                                     const int* nseg, int n_total, int k_total, int b_rows_per_slot,
                                     __nv_bfloat16* out, int out_ld, int num_ctas, cudaStream_t stream) {
  if (n_total % BN || k_total % BK) return cudaErrorInvalidValue;
  if (epi == EPI_SWIGLU)
    grouped_gemm_m256_kernel<EPI_SWIGLU><<<num_ctas, kThreads, kSmemBytes4, stream>>>(
        *tmA, *tmB, segs, nseg, n_total, k_total, b_rows_per_slot, out, out_ld);
  else
    grouped_gemm_m256_kernel<EPI_STORE><<<num_ctas, kThreads, kSmemBytes4, stream>>>(
        *tmA, *tmB, segs, nseg, n_total, k_total, b_rows_per_slot, out, out_ld);
  return cudaGetLastError();
}

// ===================================================================
// Swap-AB decode variant: in the decode regime (a few to a few dozen rows per
// replica) the 128-row token tile of the kernels above is mostly padding, so
// the tensor pipe multiplies every weight byte by 128 rows while the kernel is
// bound by the weight stream.  Here the WEIGHTS are the M operand (two M=128
// halves of the 256-row weight tile, K-major, the same TMA boxes) and the
// tokens are N: one tile = up to SN = 64 rows of one segment, the MMA's N set
// per tile to the rows rounded up to 16 (runtime instruction descriptor).
// D[feature][token] lands in TMEM with features on the lanes; the epilogue
// pairs neighbouring lanes (shfl) so each thread stores two adjacent bf16
// features of one token.  Per weight byte the tensor work drops from 128 rows
// to the rows actually present, and the smem stage is 32 KB of weights + 4-8
// KB of tokens (5 stages).
// SN = 64 (decode: 5 stages of 32 KB weights + 8 KB tokens) or 128 (mid-size
// batches: the 1-SM kernel's MMA work per stage, 4 stages of 48 KB, plus the
// fused GEMM1 -> GEMM2 schedule).
constexpr int SBOX = 32;
constexpr uint32_t kStageWS = BN * BK * 2, kBoxBytesS = SBOX * BK * 2;
template <int SN_>
struct SwapCfg {
  static constexpr int SN = SN_;
  static constexpr int STAGES = SN_ == 64 ? 5 : 4;
  static constexpr uint32_t kStageTok = SN_ * BK * 2;
  static constexpr uint32_t kTmemCols = 4 * SN_;  // 2 accumulators x 2 weight halves x SN token columns
  // smem layout, offsets relative to the 1024-aligned base
  static constexpr uint32_t a = 0;  // token tiles
  static constexpr uint32_t b = a + STAGES * kStageTok;
  static constexpr uint32_t bars = b + STAGES * kStageWS;
  static constexpr uint32_t n_bars = 2 * STAGES + 4 + 2 * kTileRing;
  static constexpr uint32_t tmem_slot = bars + n_bars * 8;
  static constexpr uint32_t tile_ring = tmem_slot + 16;              // int[kTileRing] (FUSED: claimed tiles)
  static constexpr uint32_t mt_prefix = tile_ring + kTileRing * 4;   // int[kMaxSegs + 1]: m-tiles before segment s
  static constexpr uint32_t segs = mt_prefix + (kMaxSegs + 1) * 4 + 12;
  static constexpr uint32_t end = ((segs + 15) / 16) * 16 + kMaxSegs * 16;
  static constexpr uint32_t kSmemBytes = end + 1024;
  static_assert(kSmemBytes <= 232448, "smem budget (swap-AB variant)");
};
// SN-row m-tiles swept per n column
__host__ __device__ constexpr int group_ms(int epi, int sn) { return (epi == 0 ? 64 : 32) * 64 / sn; }

// 32 token columns of one accumulator half -> bf16 pairs of features:
// lane pairs (2i, 2i+1) swap one value so the even lane stores token j's
// features (f, f+1) and the odd lane token j+1's.
__device__ __forceinline__ void store_token_pairs(const float (&v)[32], int lane, int j0, int rows,
                                                  __nv_bfloat16* __restrict__ base, size_t row0, int out_ld,
                                                  int col_even) {
  const bool odd = lane & 1;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const float a = v[2 * i], b = v[2 * i + 1];  // tokens j0+2i, j0+2i+1 of this lane's feature
    const float other = __shfl_xor_sync(0xffffffffu, odd ? a : b, 1);
    const int row = j0 + 2 * i + (odd ? 1 : 0);
    const uint32_t packed = odd ? pack_bf16(other, b) : pack_bf16(a, other);
    if (row < rows) *reinterpret_cast<uint32_t*>(base + (row0 + row) * out_ld + col_even) = packed;
  }
}

// One GEMM of the swap kernel: GEMM1 (SwiGLU into H) or GEMM2 (store Yp).
struct SwapPass {
  __nv_bfloat16* out;
  int n_tiles, num_kb, b_rows_per_slot, out_ld, epi;
  int wrows;  // weight rows per tile: 256 (two M=128 halves), or 128 for GEMM2 (half tiles: a shorter tail)
};

struct SwapTile {
  int pass, seg, m, n;
};

// tile t of the launch -> (pass, segment, m-tile, n-tile); the tiles of pass 0
// come first, each pass in decode_tile's grouped order
template <int SN>
__device__ __forceinline__ SwapTile swap_tile(int t, const int* mt_prefix, int nseg, int mt_total,
                                              const SwapPass& p0, const SwapPass& p1) {
  SwapTile r;
  r.pass = t >= mt_total * p0.n_tiles ? 1 : 0;
  const SwapPass& p = r.pass ? p1 : p0;
  if (r.pass) t -= mt_total * p0.n_tiles;
  int lo = 0, hi = nseg - 1;  // last s with mt_prefix[s] * n_tiles <= t
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (mt_prefix[mid] * p.n_tiles <= t) lo = mid; else hi = mid - 1;
  }
  r.seg = lo;
  const int local = t - mt_prefix[lo] * p.n_tiles;
  const int m_tiles = mt_prefix[lo + 1] - mt_prefix[lo];
  const int GM = group_ms(p.epi, SN);
  const int per_group = GM * p.n_tiles;
  const int g = local / per_group;
  const int gm = min(GM, m_tiles - g * GM);
  const int rem = local - g * per_group;
  r.n = rem / gm;
  r.m = g * GM + rem % gm;
  return r;
}

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// FUSED: one launch runs GEMM1 then GEMM2 (pass 0 / pass 1).  A GEMM2 tile of
// (segment, m-tile) waits, before loading its H rows, until every GEMM1 tile
// of those rows has been stored: ready[(segment, m-tile)] counts epilogue
// warps done (4 per GEMM1 n-tile).  Tiles are CLAIMED in order from a global
// counter (the producer hands each claim to the MMA and epilogue warps through
// a shared-memory ring), so when a GEMM2 tile is claimed every GEMM1 tile has
// already been claimed by a running CTA that finishes it without waiting on
// anything: no deadlock even when the grid is not fully resident (other
// kernels on the GPU).  The last CTA to finish zeroes the counters.  GEMM2's weights start streaming while GEMM1's
// last wave drains, and there is no tail between the two GEMMs.
// MOE_FRONT_TRACE: %globaltimer at each swap-kernel CTA's start / end ([cta][12], [cta][13] of the trace)
__device__ unsigned long long* g_swap_trace = nullptr;
__device__ __forceinline__ void swap_stamp(int i) {
  unsigned long long* tr = g_swap_trace;
  if (tr && threadIdx.x == 0) {
    unsigned long long v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    tr[blockIdx.x * 16 + i] = v;
  }
}
cudaError_t set_swap_trace(unsigned long long* p) { return cudaMemcpyToSymbol(g_swap_trace, &p, sizeof(p)); }

template <bool FUSED, int SNv>
__global__ void __launch_bounds__(kThreads, 1)
grouped_gemm_swap_kernel(const __grid_constant__ CUtensorMap tmA0, const __grid_constant__ CUtensorMap tmB0,
                         const __grid_constant__ CUtensorMap tmA1, const __grid_constant__ CUtensorMap tmB1,
                         const GemmSeg* __restrict__ segs_g, const int* __restrict__ nseg_g, const SwapPass p0,
                         const SwapPass p1, int* __restrict__ ready, int ready_n, int wpol) {
  using C = SwapCfg<SNv>;
  constexpr int SN = C::SN, STAGES_S = C::STAGES;
  constexpr uint32_t kStageTokS = C::kStageTok;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::bars);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES_S;
  uint64_t* tfull = bars + 2 * STAGES_S;
  uint64_t* tempty = bars + 2 * STAGES_S + 2;
  uint64_t* ring_full = bars + 2 * STAGES_S + 4;
  uint64_t* ring_empty = ring_full + kTileRing;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::tmem_slot);
  volatile int* ring = reinterpret_cast<volatile int*>(smem + C::tile_ring);
  int* mt_prefix = reinterpret_cast<int*>(smem + C::mt_prefix);
  int* claim = ready + ready_n - 2;  // FUSED: next tile to claim
  int4* segs = reinterpret_cast<int4*>(smem + C::segs);

  const int warp = threadIdx.x >> 5;
  const int lane = lane_id();
  swap_stamp(12);
  const int nseg = min(*nseg_g, kMaxSegs);

  for (int i = threadIdx.x; i < nseg; i += kThreads) segs[i] = reinterpret_cast<const int4*>(segs_g)[i];
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA0);
    tma_prefetch_desc(&tmB0);
    if (FUSED) {
      tma_prefetch_desc(&tmA1);
      tma_prefetch_desc(&tmB1);
    }
    for (int s = 0; s < STAGES_S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 4); }
    for (int r = 0; r < kTileRing; ++r) { mbar_init(&ring_full[r], 1); mbar_init(&ring_empty[r], 5); }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<C::kTmemCols>(tmem_slot);
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int s = 0; s < nseg; ++s) {
      mt_prefix[s] = acc;
      acc += (segs[s].y + SN - 1) / SN;
    }
    mt_prefix[nseg] = acc;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int mt_total = nseg > 0 ? mt_prefix[nseg] : 0;
  const int total_tiles = mt_total * (p0.n_tiles + (FUSED ? p1.n_tiles : 0));
  const int ready_target = 4 * p0.n_tiles;
  griddep_launch_dependents();

  if (warp == 0) {
    // ---------------------------------------------------------- producer
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      const uint64_t pol_b = wpol == 1 ? policy_evict_first() : (wpol == 2 ? policy_evict_normal() : policy_evict_last());
      bool first = true;
      int rslot = 0;
      uint32_t rphase = 0;
      for (int t = blockIdx.x;; t += gridDim.x) {
        if (FUSED) {
          t = atomicAdd(claim, 1);
          mbar_wait(&ring_empty[rslot], rphase ^ 1);
          ring[rslot] = t < total_tiles ? t : -1;
          mbar_arrive(&ring_full[rslot]);
          if (++rslot == kTileRing) { rslot = 0; rphase ^= 1; }
        }
        if (t >= total_tiles) break;
        const SwapTile c = swap_tile<SN>(t, mt_prefix, nseg, mt_total, p0, p1);
        const SwapPass& p = c.pass ? p1 : p0;
        const CUtensorMap* tA = c.pass ? &tmA1 : &tmA0;
        const CUtensorMap* tB = c.pass ? &tmB1 : &tmB0;
        const int a_row = segs[c.seg].x + c.m * SN;
        const int rows = min(SN, segs[c.seg].y - c.m * SN);
        const int nbox = (rows + SBOX - 1) / SBOX;
        const uint32_t bytes = p.wrows * BK * 2 + nbox * kBoxBytesS;
        const int b_row = segs[c.seg].z * p.b_rows_per_slot + c.n * p.wrows;
        const int num_kb = p.num_kb;
        int kb0 = 0;
        if (first || (FUSED && c.pass == 1)) {
          // Weights of the first stages go first: they depend neither on the
          // producer kernel (PDL) nor on the GEMM1 tiles of these rows.
          kb0 = num_kb < STAGES_S ? num_kb : STAGES_S;
          const int st0 = stage;
          for (int kb = 0; kb < kb0; ++kb) {
            if (!first) mbar_wait(&empty[stage], phase ^ 1);  // fresh stages need no wait
            mbar_arrive_expect_tx(&full[stage], bytes);
            tma_load_2d_hint(smem + C::b + stage * kStageWS, tB, &full[stage], kb * BK, b_row, pol_b);
            if (++stage == STAGES_S) { stage = 0; phase ^= 1; }
          }
          if (first) griddep_wait();
          first = false;
          if (FUSED && c.pass == 1) {
            const int* r = ready + mt_prefix[c.seg] + c.m;
            while (ld_acquire_gpu(r) < ready_target) __nanosleep(100);
            fence_proxy_async_global();  // H was written by generic stores of other SMs
          }
          int st = st0;
          for (int kb = 0; kb < kb0; ++kb) {
            for (int bx = 0; bx < nbox; ++bx)
              tma_load_2d(smem + C::a + st * kStageTokS + bx * kBoxBytesS, tA, &full[st], kb * BK,
                          a_row + bx * SBOX);
            if (++st == STAGES_S) st = 0;
          }
        }
        for (int kb = kb0; kb < num_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], bytes);
          tma_load_2d_hint(smem + C::b + stage * kStageWS, tB, &full[stage], kb * BK, b_row, pol_b);
          for (int bx = 0; bx < nbox; ++bx)
            tma_load_2d(smem + C::a + stage * kStageTokS + bx * kBoxBytesS, tA, &full[stage], kb * BK,
                        a_row + bx * SBOX);
          if (++stage == STAGES_S) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------- MMA issuer
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      const uint32_t a_base = smem_u32(smem + C::a);
      const uint32_t b_base = smem_u32(smem + C::b);
      int rslot = 0;
      uint32_t rphase = 0;
      for (int t = blockIdx.x;; t += gridDim.x) {
        if (FUSED) {
          mbar_wait(&ring_full[rslot], rphase);
          t = ring[rslot];
          mbar_arrive(&ring_empty[rslot]);
          if (++rslot == kTileRing) { rslot = 0; rphase ^= 1; }
          if (t < 0) break;
        } else if (t >= total_tiles) {
          break;
        }
        const SwapTile c = swap_tile<SN>(t, mt_prefix, nseg, mt_total, p0, p1);
        const int num_kb = (c.pass ? p1 : p0).num_kb;
        const bool two_halves = (c.pass ? p1 : p0).wrows == 256;
        const int rows = min(SN, segs[c.seg].y - c.m * SN);
        const uint32_t idesc = umma_idesc_bf16(128, static_cast<uint32_t>((rows + 15) & ~15));
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d0 = tmem_base + acc * 2 * SN, d1 = d0 + SN;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t w_st = b_base + stage * kStageWS;
          const uint64_t w_top = umma_desc_sw128(w_st);
          const uint64_t w_bot = umma_desc_sw128(w_st + 128 * 128);  // weight rows 128..255: +16 KB
          const uint64_t tdesc = umma_desc_sw128(a_base + stage * kStageTokS);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint32_t accf = (kb | k) != 0 ? 1u : 0u;
            tc_mma_bf16(d0, w_top + 2 * k, tdesc + 2 * k, idesc, accf);
            if (two_halves) tc_mma_bf16(d1, w_bot + 2 * k, tdesc + 2 * k, idesc, accf);
          }
          tc_commit(&empty[stage]);
          if (++stage == STAGES_S) { stage = 0; phase ^= 1; }
        }
        tc_commit(&tfull[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    // --------------------------------------------------------- epilogue
    const int quarter = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    int rslot = 0;
    uint32_t rphase = 0;
    for (int t = blockIdx.x;; t += gridDim.x) {
      if (FUSED) {
        mbar_wait(&ring_full[rslot], rphase);
        t = ring[rslot];
        __syncwarp();
        if (lane == 0) mbar_arrive(&ring_empty[rslot]);
        if (++rslot == kTileRing) { rslot = 0; rphase ^= 1; }
        if (t < 0) break;
      } else if (t >= total_tiles) {
        break;
      }
      const SwapTile c = swap_tile<SN>(t, mt_prefix, nseg, mt_total, p0, p1);
      const SwapPass& p = c.pass ? p1 : p0;
      const int4 sg = segs[c.seg];
      const int rows = min(SN, sg.y - c.m * SN);
      const size_t row0 = static_cast<size_t>(sg.x) + c.m * SN;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + acc * 2 * SN;
      const int f = quarter * 32 + lane;  // this thread's feature within a 128-row weight half
#pragma unroll 1
      for (int j0 = 0; j0 < rows; j0 += 32) {
        float v[32];
        if (p.epi == EPI_SWIGLU) {
          uint32_t g[32], u[32];
          tmem_ld_32x32b_x32(taddr + j0, g);       // W1 half: gate projections
          tmem_ld_32x32b_x32(taddr + SN + j0, u);  // W3 half: up projections
          tc_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = silu(__uint_as_float(g[i])) * __uint_as_float(u[i]);
          store_token_pairs(v, lane, j0, rows, p.out, row0, p.out_ld, c.n * (BN / 2) + (f & ~1));
        } else {
#pragma unroll 1
          for (int h = 0; h < p.wrows / 128; ++h) {
            uint32_t r[32];
            tmem_ld_32x32b_x32(taddr + h * SN + j0, r);
            tc_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
            store_token_pairs(v, lane, j0, rows, p.out, row0, p.out_ld, c.n * p.wrows + h * 128 + (f & ~1));
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      if (FUSED && c.pass == 0) {
        // this warp's share of the tile's H rows is stored: publish it
        fence_proxy_async_global();
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicAdd(ready + mt_prefix[c.seg] + c.m, 1);
      }
    }
  }
  griddep_wait();
  tc_fence_before();
  __syncthreads();
  if (FUSED && threadIdx.x == 0) {
    // every tile of this CTA is done; the last CTA resets the counters
    __threadfence();
    if (atomicAdd(ready + ready_n - 1, 1) == static_cast<int>(gridDim.x) - 1) {
      for (int i = 0; i < mt_total; ++i) ready[i] = 0;
      *claim = 0;
      ready[ready_n - 1] = 0;
      __threadfence();
    }
  }
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::kTmemCols>(tmem_base);
  }
  swap_stamp(13);
}

std::atomic<int> g_gemm_l2pol{-1};  // 2-SM K4 L2 policies (env MOE_GEMM_L2POL: GEMM1 bits 0-3, GEMM2 bits 4-7; -1 default)
std::atomic<int> g_swap_wpol{1};  // L2 policy of the swap kernel's weight stream: 1 evict_first (default), 0 evict_last, 2 normal (env MOE_SWAP_WPOL)

template <int SNv>
cudaError_t launch_swap(int which, const CUtensorMap* tmA1, const CUtensorMap* tmB1, const CUtensorMap* tmA2,
                        const CUtensorMap* tmB2, const GemmSeg* segs, const int* nseg, const SwapPass& g1,
                        const SwapPass& g2, int* ready, int ready_n, int num_ctas, cudaStream_t stream, bool pdl) {
  using C = SwapCfg<SNv>;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(num_ctas);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = C::kSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (which == 2)
    return cudaLaunchKernelEx(&cfg, grouped_gemm_swap_kernel<true, SNv>, *tmA1, *tmB1, *tmA2, *tmB2, segs, nseg, g1,
                              g2, ready, ready_n, g_swap_wpol.load(std::memory_order_relaxed));
  if (which == 0)
    return cudaLaunchKernelEx(&cfg, grouped_gemm_swap_kernel<false, SNv>, *tmA1, *tmB1, *tmA1, *tmB1, segs, nseg,
                              g1, g1, ready, ready_n, g_swap_wpol.load(std::memory_order_relaxed));
  return cudaLaunchKernelEx(&cfg, grouped_gemm_swap_kernel<false, SNv>, *tmA2, *tmB2, *tmA2, *tmB2, segs, nseg, g2,
                            g2, ready, ready_n, g_swap_wpol.load(std::memory_order_relaxed));
}

// which: 0 = GEMM1 alone, 1 = GEMM2 alone, 2 = GEMM1 then GEMM2 in one launch;
// sn = token rows per tile (64 or 128).
cudaError_t launch_grouped_gemm_swap(int which, int sn, const CUtensorMap* tmA1, const CUtensorMap* tmB1,
                                     const CUtensorMap* tmA2, const CUtensorMap* tmB2, const GemmSeg* segs,
                                     const int* nseg, int d, int ff, int b_rows1, int b_rows2, __nv_bfloat16* h,
                                     __nv_bfloat16* yp, int* ready, int ready_n, int num_ctas, cudaStream_t stream,
                                     bool pdl, const CUtensorMap* tmB2half) {
  if ((2 * ff) % BN || d % BN || d % BK || ff % BK || (sn != 64 && sn != 128)) return cudaErrorInvalidValue;
  const int w2rows = tmB2half ? 128 : 256;
  const SwapPass g1{h, 2 * ff / BN, d / BK, b_rows1, ff, EPI_SWIGLU, 256};
  const SwapPass g2{yp, d / w2rows, ff / BK, b_rows2, d, EPI_STORE, w2rows};
  if (tmB2half) tmB2 = tmB2half;
  return sn == 64 ? launch_swap<64>(which, tmA1, tmB1, tmA2, tmB2, segs, nseg, g1, g2, ready, ready_n, num_ctas,
                                    stream, pdl)
                  : launch_swap<128>(which, tmA1, tmB1, tmA2, tmB2, segs, nseg, g1, g2, ready, ready_n, num_ctas,
                                     stream, pdl);
}

// --------------------------------------------------------------- host side
static_assert(kSmemBytes <= 232448, "smem budget");

cudaError_t launch_grouped_gemm_2sm(int epi, const CUtensorMap* tmA, const CUtensorMap* tmB, const GemmSeg* segs,
                                    const int* nseg, int n_total, int k_total, int b_rows_per_slot,
                                    __nv_bfloat16* out, int out_ld, int num_ctas, cudaStream_t stream, bool pdl,
                                    int group_m, int* sched, const int32_t* fy_row_owner, const float* fy_wts,
                                    __nv_bfloat16* fy_y, int32_t* fy_cnt) {
  const FusedY fy{fy_y ? fy_row_owner : nullptr, fy_wts, fy_y, fy_cnt, n_total, n_total / BN};
  if (n_total % BN || k_total % BK) return cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(num_ctas & ~1);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemBytes2;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const int gp = group_m > 0 ? (group_m + 1) / 2 : 0;  // m-tiles -> 256-row tiles
  const int pol = g_gemm_l2pol.load(std::memory_order_relaxed);
  const int l2pol = pol >= 0 ? (epi == EPI_SWIGLU ? pol & 15 : (pol >> 4) & 15) : 1 << 2;
  if (epi == EPI_SWIGLU)
    return cudaLaunchKernelEx(&cfg, grouped_gemm_2sm_kernel<EPI_SWIGLU>, *tmA, *tmB, segs, nseg, n_total, k_total,
                              b_rows_per_slot, out, out_ld, gp, l2pol, sched, FusedY{});
  return cudaLaunchKernelEx(&cfg, grouped_gemm_2sm_kernel<EPI_STORE>, *tmA, *tmB, segs, nseg, n_total, k_total,
                            b_rows_per_slot, out, out_ld, gp, l2pol, sched, fy);
}

cudaError_t launch_grouped_gemm_mc(int epi, const CUtensorMap* tmA, const CUtensorMap* tmBh, const GemmSeg* segs,
                                   const int* nseg, int n_total, int k_total, int b_rows_per_slot,
                                   __nv_bfloat16* out, int out_ld, int num_ctas, cudaStream_t stream, bool pdl,
                                   int group_m) {
  if (n_total % BN || k_total % BK) return cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(num_ctas & ~1);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // group_m counts m-tiles; the kernel sweeps pairs of them
  const int gp = group_m > 0 ? (group_m + 1) / 2 : 0;
  if (epi == EPI_SWIGLU)
    return cudaLaunchKernelEx(&cfg, grouped_gemm_mc_kernel<EPI_SWIGLU>, *tmA, *tmBh, segs, nseg, n_total, k_total,
                              b_rows_per_slot, out, out_ld, gp);
  return cudaLaunchKernelEx(&cfg, grouped_gemm_mc_kernel<EPI_STORE>, *tmA, *tmBh, segs, nseg, n_total, k_total,
                            b_rows_per_slot, out, out_ld, gp);
}

int gemm_smem_bytes() { return static_cast<int>(kSmemBytes); }

cudaError_t launch_grouped_gemm(int epi, const CUtensorMap* tmA, const CUtensorMap* tmB, const GemmSeg* segs,
                                const int* nseg, int n_total, int k_total, int b_rows_per_slot,
                                __nv_bfloat16* out, int out_ld, int num_ctas, cudaStream_t stream, int* sched,
                                bool pdl, const int32_t* a_gather, int group_m, const FusedCombine& fc) {
  if (n_total % BN || k_total % BK) return cudaErrorInvalidValue;
  // programmatic dependent launch: the kernel starts while the previous one
  // drains (it waits in griddepcontrol.wait before reading A)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(num_ctas);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (epi == EPI_SWIGLU)
    return cudaLaunchKernelEx(&cfg, grouped_gemm_kernel<EPI_SWIGLU>, *tmA, *tmB, segs, nseg, n_total, k_total,
                              b_rows_per_slot, out, out_ld, sched, a_gather, group_m, fc);
  return cudaLaunchKernelEx(&cfg, grouped_gemm_kernel<EPI_STORE>, *tmA, *tmB, segs, nseg, n_total, k_total,
                            b_rows_per_slot, out, out_ld, sched, a_gather, group_m, fc);
}

// Load every kernel of this file now (CUDA 12 loads kernels lazily on first
// launch, and a lazy load may wait for the whole context — including a
// peer-exchange kernel spinning on another rank that shares the context).
//
// Also sets the dynamic shared-memory opt-in of every K4 kernel.  The
// attribute is per device, so this runs for every context after its
// cudaSetDevice (moe_ctx_create), not once per process.
cudaError_t preload_gemm_kernels() {
  const struct {
    const void* fn;
    size_t smem;
  } opt_in[] = {{reinterpret_cast<const void*>(grouped_gemm_kernel<EPI_SWIGLU>), kSmemBytes},
                {reinterpret_cast<const void*>(grouped_gemm_kernel<EPI_STORE>), kSmemBytes},
                {reinterpret_cast<const void*>(grouped_gemm_mc_kernel<EPI_SWIGLU>), kSmemBytes},
                {reinterpret_cast<const void*>(grouped_gemm_mc_kernel<EPI_STORE>), kSmemBytes},
                {reinterpret_cast<const void*>(grouped_gemm_2sm_kernel<EPI_SWIGLU>), kSmemBytes2},
                {reinterpret_cast<const void*>(grouped_gemm_2sm_kernel<EPI_STORE>), kSmemBytes2},
                {reinterpret_cast<const void*>(grouped_gemm_m256_kernel<EPI_SWIGLU>), kSmemBytes4},
                {reinterpret_cast<const void*>(grouped_gemm_m256_kernel<EPI_STORE>), kSmemBytes4},
                {reinterpret_cast<const void*>(grouped_gemm_swap_kernel<false, 64>), SwapCfg<64>::kSmemBytes},
                {reinterpret_cast<const void*>(grouped_gemm_swap_kernel<true, 64>), SwapCfg<64>::kSmemBytes},
                {reinterpret_cast<const void*>(grouped_gemm_swap_kernel<false, 128>), SwapCfg<128>::kSmemBytes},
                {reinterpret_cast<const void*>(grouped_gemm_swap_kernel<true, 128>), SwapCfg<128>::kSmemBytes}};
  for (const auto& k : opt_in) {
    const cudaError_t e =
        cudaFuncSetAttribute(k.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(k.smem));
    if (e != cudaSuccess) return e;
  }
  cudaFuncAttributes a;
  const void* fns[] = {reinterpret_cast<const void*>(grouped_gemm_kernel<0>),
                       reinterpret_cast<const void*>(grouped_gemm_kernel<1>),
                       reinterpret_cast<const void*>(grouped_gemm_2sm_kernel<0>),
                       reinterpret_cast<const void*>(grouped_gemm_2sm_kernel<1>),
                       reinterpret_cast<const void*>(grouped_gemm_m256_kernel<0>),
                       reinterpret_cast<const void*>(grouped_gemm_m256_kernel<1>),
                       reinterpret_cast<const void*>(grouped_gemm_swap_kernel<false, 64>),
                       reinterpret_cast<const void*>(grouped_gemm_swap_kernel<true, 64>),
                       reinterpret_cast<const void*>(grouped_gemm_swap_kernel<false, 128>),
                       reinterpret_cast<const void*>(grouped_gemm_swap_kernel<true, 128>)};
  for (const void* f : fns) {
    const cudaError_t e = cudaFuncGetAttributes(&a, f);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace moe
