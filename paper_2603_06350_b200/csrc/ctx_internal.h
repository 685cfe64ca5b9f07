// ctx_internal.h — the per-device context behind the C-ABI (include/moe_b200.h):
// kernel launcher declarations, device buffers, per-layer state (weight pools,
// placement, residency, predictor bookkeeping) and struct moe_ctx, shared by
// capi_ctx.cpp (context, weights, placement, residency) and capi.cpp (the
// forward: gate -> plan -> dispatch -> K4 -> combine).  Internal: not installed.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <tuple>
#include <stdexcept>
#include <unistd.h>
#include <string>
#include <vector>

#include "capi_util.h"
#include "host/exchange_plan.h"
#include "kernels/dispatch_plan.h"
#include "moe_b200.h"
#include "transport.h"
#include "host/moeless_api.hpp"

namespace moe {
// kernels
int gate_num_blocks(int T);
cudaError_t launch_gate_topk(const __nv_bfloat16* x, int T, int d, const __nv_bfloat16* w_all, int E, int n_pred,
                             int k, int32_t* ids, float* wts, int32_t* counts, int32_t* block_counts,
                             int32_t* pred_counts, float* partial, cudaStream_t stream,
                             int32_t* host_counts = nullptr, int host_n = 0, unsigned* ticket = nullptr,
                             const float* pred_w2 = nullptr, unsigned mlp_mask = 0,
                             const CUtensorMap* tmx = nullptr);
cudaError_t launch_route_ids(const int32_t* ids_in, const float* w_in, int T, int E, int k, int32_t* ids, float* wts,
                             int32_t* counts, int32_t* block_counts, int* err, cudaStream_t s);
cudaError_t launch_block_prefix(const int32_t* block_counts, int nblk, int E, const DevPlan* plan,
                                int32_t* block_pre, cudaStream_t s, const int32_t* local_counts = nullptr,
                                bool pdl = false);
cudaError_t launch_dispatch(const __nv_bfloat16* x, int T, int d, int E, int k, const int32_t* ids,
                            const int32_t* block_pre, const DevPlan* plan, const RowTargets& targets,
                            uint32_t* row_code, const PeerSignal& sig, cudaStream_t s, int32_t* perm_src,
                            int32_t* row_owner, bool pdl = false, const int32_t* local_counts = nullptr,
                            const int32_t* block_counts = nullptr, DevPlan* plan_out = nullptr);
bool dispatch_fuses_plan(int T);  // single GPU: dispatch builds prefix + plan itself (few blocks)
// decode front end in one cooperative launch (kernels/frontend.cu): gate + top-k + plan + dispatch
bool frontend_applies(int T, int d, int Etot, int k, int num_sms);
cudaError_t launch_frontend(const __nv_bfloat16* x, int T, int d, const __nv_bfloat16* w_all, int E, int n_pred, int k,
                            int32_t* ids, float* wts, int32_t* counts, int32_t* block_counts, float* partial,
                            int32_t* host_counts, const float* pred_w2, unsigned mlp_mask, __nv_bfloat16* xp,
                            uint32_t* row_code, DevPlan* plan, const void* prefetch, size_t prefetch_bytes,
                            unsigned long long* trace, cudaStream_t stream);
cudaError_t preload_frontend_kernels();
cudaError_t set_swap_trace(unsigned long long* p);
cudaError_t set_combine_trace(unsigned long long* p);
cudaError_t launch_trace_marker(cudaStream_t s);  // MOE_FRONT_TRACE: swap-AB K4 CTA start / end stamps
// prefill gate on tcgen05 (kernels/gate.cu): 128-token tiles, TMA-streamed x
bool gate_tc_applies(int T, int d, int Etot, int k, bool mlp);
cudaError_t launch_gate_tc(const CUtensorMap* tmx, const CUtensorMap* tmw, int T, int d, int E, int n_pred, int k,
                           int32_t* ids, float* wts, int32_t* counts, int32_t* block_counts, int32_t* pred_counts,
                           int32_t* host_counts, int host_n, unsigned* ticket, int num_sms, cudaStream_t stream,
                           unsigned long long* trace = nullptr);
extern std::atomic<int> g_gate_tc, g_gate_tc_bks;
// K6 over peer memory (p2p.cu)
constexpr int kMaxRanks = 8;
enum { kFlagCounts = 0, kFlagRows = 1, kFlagOutputs = 2, kFlagKinds = 4 };
struct PeerSlabs {
  uint32_t* flags[kMaxRanks];
  const int32_t* counts[kMaxRanks];
};
cudaError_t launch_p2p_signal(const PeerSlabs& peers, int G, int kind, int src, const uint32_t* epoch,
                              cudaStream_t s);
cudaError_t launch_p2p_wait(const uint32_t* my_flags, int G, int kind, const uint32_t* epoch, uint64_t timeout_ns,
                            int* err, cudaStream_t s);
cudaError_t launch_p2p_counts(const PeerSlabs& peers, int G, int rank, int stride, uint32_t* epoch,
                              uint64_t timeout_ns, int* err, int32_t* counts_all, cudaStream_t s);
cudaError_t launch_small_copy(void* dst, const void* src, size_t bytes, cudaStream_t s);
cudaError_t launch_l2_prefetch(const void* base, size_t bytes, cudaStream_t s);
cudaError_t launch_plan_exchange(const int32_t* counts_all, int stride, int G, int rank, const PlacementTable* pt,
                                 DevPlan* plan, cudaStream_t s);
// K7 fp32 path
cudaError_t launch_gate_f32(const float* x, int T, int d, const float* wg, int E, int k, int32_t* ids, float* wts,
                            int32_t* counts, int32_t* block_counts, cudaStream_t s);
cudaError_t launch_grouped_sgemm(const float* A, int lda, const float* Bpool, int b_rows_per_slot, int ldb,
                                 const GemmSeg* segs, const int* nseg, int N, int K, float* C, int ldc, int num_sms,
                                 cudaStream_t s);
cudaError_t launch_swiglu_f32(const float* C, int rows, int ff, float* H, cudaStream_t s);
cudaError_t launch_combine_f32(const RowTargets& sources, int T, int d, int k, const uint32_t* row_code,
                               const float* wts, float* y, cudaStream_t s);
cudaError_t launch_combine(const RowTargets& sources, int T, int d, int k, const uint32_t* row_code,
                           const float* wts, __nv_bfloat16* y, int num_sms, cudaStream_t s, bool pdl = false);
cudaError_t launch_grouped_gemm_m256(int epi, const CUtensorMap* tmA, const CUtensorMap* tmB, const GemmSeg* segs,
                                     const int* nseg, int n_total, int k_total, int b_rows_per_slot,
                                     __nv_bfloat16* out, int out_ld, int num_ctas, cudaStream_t stream);
cudaError_t launch_grouped_gemm_2sm(int epi, const CUtensorMap* tmA, const CUtensorMap* tmB, const GemmSeg* segs,
                                    const int* nseg, int n_total, int k_total, int b_rows_per_slot,
                                    __nv_bfloat16* out, int out_ld, int num_ctas, cudaStream_t stream, bool pdl = false,
                                    int group_m = 0, int* sched = nullptr, const int32_t* fy_row_owner = nullptr,
                                    const float* fy_wts = nullptr, __nv_bfloat16* fy_y = nullptr,
                                    int32_t* fy_cnt = nullptr);
cudaError_t launch_grouped_gemm_mc(int epi, const CUtensorMap* tmA, const CUtensorMap* tmBh, const GemmSeg* segs,
                                   const int* nseg, int n_total, int k_total, int b_rows_per_slot,
                                   __nv_bfloat16* out, int out_ld, int num_ctas, cudaStream_t stream, bool pdl,
                                   int group_m);
cudaError_t launch_grouped_gemm(int epi, const CUtensorMap* tmA, const CUtensorMap* tmB, const GemmSeg* segs,
                                const int* nseg, int n_total, int k_total, int b_rows_per_slot,
                                __nv_bfloat16* out, int out_ld, int num_ctas, cudaStream_t stream, int* sched,
                                bool pdl, const int32_t* a_gather, int group_m, const FusedCombine& fc);
cudaError_t launch_grouped_gemm_swap(int which, int sn, const CUtensorMap* tmA1, const CUtensorMap* tmB1,
                                     const CUtensorMap* tmA2, const CUtensorMap* tmB2, const GemmSeg* segs,
                                     const int* nseg, int d, int ff, int b_rows1, int b_rows2, __nv_bfloat16* h,
                                     __nv_bfloat16* yp, int* ready, int ready_n, int num_ctas, cudaStream_t stream,
                                     bool pdl, const CUtensorMap* tmB2half = nullptr);
extern std::atomic<int> g_gate_max_splits;  // K1 split-K bound (env MOE_GATE_MAX_SPLITS)
extern std::atomic<int> g_gate_cluster;     // K1 split-K reduced in a cluster (env MOE_GATE_CLUSTER)
extern std::atomic<int> g_gate_min_splits;  // K1 split-K floor (env MOE_GATE_MIN_SPLITS)
extern std::atomic<int> g_gate_stream;      // K1 persistent streaming kernel for large batches (env MOE_GATE_STREAM)
extern std::atomic<int> g_gemm_l2pol;  // 2-SM K4 L2 policies (env MOE_GEMM_L2POL)
extern std::atomic<int> g_swap_wpol;  // swap-AB weight-stream L2 policy (env MOE_SWAP_WPOL)
cudaError_t preload_gate_kernels();
cudaError_t preload_dispatch_kernels();
cudaError_t preload_gemm_kernels();
cudaError_t preload_fp32_kernels();
cudaError_t preload_p2p_kernels();
// host
uint64_t stream_key(uint64_t seed, uint64_t a, uint64_t b, uint64_t tag);
void synth_tokens(uint64_t key, int64_t first, int64_t tokens, int d, int E, uint16_t* x);
void synth_gate(uint64_t key, int d, int E, const double* pop, const int32_t* noise_perm, uint16_t* wg);
void synth_expert(uint64_t key, int d, int ff, uint16_t* w1, uint16_t* w3, uint16_t* w2);
}  // namespace moe

using namespace moe;

// ====================================================================== errors
namespace moe {

#define CU_CHECK(expr)                                                                      \
  do {                                                                                      \
    cudaError_t _e = (expr);                                                                \
    if (_e != cudaSuccess)                                                                  \
      throw Status(MOE_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));          \
  } while (0)

static_assert(sizeof(DevPlan) % 16 == 0, "DevPlan is copied in 16-byte words");
static_assert(sizeof(PlacementTable) % 16 == 0, "PlacementTable is copied in 16-byte words");

// ======================================================================= NCCL
// Loaded lazily with dlopen so single-GPU use never depends on libnccl.
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;

  void load() {
    if (h) return;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) throw Status(MOE_ENCCL, "cannot dlopen libnccl.so.2");
    auto sym = [&](const char* s) {
      void* p = dlsym(h, s);
      if (!p) throw Status(MOE_ENCCL, std::string("libnccl lacks ") + s);
      return p;
    };
    GetUniqueId = reinterpret_cast<decltype(GetUniqueId)>(sym("ncclGetUniqueId"));
    CommInitRank = reinterpret_cast<decltype(CommInitRank)>(sym("ncclCommInitRank"));
    CommDestroy = reinterpret_cast<decltype(CommDestroy)>(sym("ncclCommDestroy"));
    AllGather = reinterpret_cast<decltype(AllGather)>(sym("ncclAllGather"));
    Send = reinterpret_cast<decltype(Send)>(sym("ncclSend"));
    Recv = reinterpret_cast<decltype(Recv)>(sym("ncclRecv"));
    GroupStart = reinterpret_cast<decltype(GroupStart)>(sym("ncclGroupStart"));
    GroupEnd = reinterpret_cast<decltype(GroupEnd)>(sym("ncclGroupEnd"));
    GetErrorString = reinterpret_cast<decltype(GetErrorString)>(sym("ncclGetErrorString"));
  }
  void check(ncclResult_t r, const char* what) const {
    if (r != ncclSuccess) throw Status(MOE_ENCCL, std::string(what) + ": " + GetErrorString(r));
  }
};
extern NcclApi g_nccl;

// ================================================================ TMA maps
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    CU_CHECK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess) throw Status(MOE_ECUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// K-major bf16 matrix [rows, cols], box = box_rows x 64 cols, 128-byte swizzle.
inline CUtensorMap make_kmajor_map(const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {cols * 2};
  const cuuint32_t box[2] = {64, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Status(MOE_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
  return m;
}

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  bool owned = true;
  void alloc(size_t count) {
    release();
    if (count) CU_CHECK(cudaMalloc(&p, count * sizeof(T)));
    n = count;
    owned = true;
  }
  void view(void* q, size_t count) {  // a window into another allocation (the P2P slab)
    release();
    p = static_cast<T*>(q);
    n = count;
    owned = false;
  }
  void release() {
    if (p && owned) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  ~DevBuf() { release(); }
};

struct Layer {
  DevBuf<uint16_t> w13, w2, wg;  // pools
  CUtensorMap tmB1, tmB2;    // 256-row boxes (1-SM kernel: whole N tile per CTA)
  CUtensorMap tmB1h, tmB2h;  // 128-row boxes (2-SM kernel: each CTA stages half of N)
  bool has_gate = false;
  std::vector<char> expert_loaded;
  std::vector<int32_t> rep_counts, rep_gpu;  // placement (host)
  bool has_placement = false;
  bool has_pred_weights = false;
  DevBuf<float> pred_w2;   // [n_pred][E][E] output layers of MLP predictor slots
  unsigned mlp_mask = 0;   // bit p: predictor slot p is an MLP (W2 set)
  // layer-aware predictor state (MOE_PLAN_PREDICTED)
  std::vector<int64_t> pred_loads;          // predicted loads for this layer (made d layers earlier)
  bool pred_valid = false;
  long plan_for = -1;                       // iteration whose placement was planned ahead
  bool boot_ready = false;                  // bootstrap placement of the next forward already planned
  double last_accuracy = -1.0, acc_sum = 0.0;
  long acc_n = 0, bootstraps = 0;
  int plan_source = 0;                      // 0 fixed, 1 actual, 2 predicted, 3 historical bootstrap
  int warm = 0, cold = 0;
  std::vector<moeless::LoadVector> history;
  // device copy of the placement for the on-device exchange planner (P2P)
  DevBuf<PlacementTable> ptab;
  PlacementTable* h_ptab = nullptr;  // pinned staging
  cudaEvent_t ev_ptab = nullptr;     // staging buffer free again
  // MOE_RESIDENCY_PLACED: which weight slot holds each expert on this rank
  std::vector<int> slot_of;           // [E], -1 = not resident
  std::vector<int> cache_expert;      // [cache slots] expert cached there, -1 free
  std::vector<long> cache_stamp;      // [cache slots] last placement that needed it (LRU)
  long placements = 0;
  std::vector<std::pair<int, int>> pending_copies;  // (slot, expert) not yet issued
  cudaEvent_t ev_used = nullptr;      // after the layer's last enqueued GEMM2 (slots free to overwrite)
  cudaEvent_t ev_wstart = nullptr, ev_wready = nullptr;  // the latest copy batch on the weight stream
  bool used_recorded = false, wready_valid = false, wready_timed = false;
  int copies_last = 0, hits_last = 0;
};

struct GraphKey {
  int layer, T;
  const void* x;
  const void* y;
  cudaEvent_t x_consumed;
  bool pred;
  unsigned mlp;  // kernel arguments captured by value: a new predictor mask is a new graph
  bool operator<(const GraphKey& o) const {
    return std::tie(layer, T, x, y, x_consumed, pred, mlp) <
           std::tie(o.layer, o.T, o.x, o.y, o.x_consumed, o.pred, o.mlp);
  }
};

struct PendingPlan {
  bool active = false;
  int layer = 0, mode = 0;
  long iteration = 0;
  int stride = 0;
  int gemm_slot = -1;  // K4 timing-ring slot whose row count the host plan fills in
};

struct EventSet {
  static constexpr int N = 10;
  cudaEvent_t ev[N] = {};
  void create() {
    for (auto& e : ev) CU_CHECK(cudaEventCreate(&e));
  }
  void destroy() {
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
  }
  float ms(int a, int b) const {
    float v = 0.0f;
    cudaEventElapsedTime(&v, ev[a], ev[b]);
    return v;
  }
};

}  // namespace moe

// =================================================================== context
struct moe_ctx {
  moe_ctx_desc desc{};
  int E = 0, k = 0, d = 0, ff = 0, G = 1, rank = 0, Tmax = 0, n_pred = 0, num_sms = 148;
  int gemm_variant = 0;  // 0 auto, 1 force 1-SM, 2 force 2-SM, 3 m256, 4 swap-AB, 5 swap64, 6 swap128, 7 mc (MOE_GEMM_VARIANT)
  int swap_rows = 64;    // auto: 64-token swap-AB tiles when the mean rows per expert <= this (MOE_GEMM_SWAP_ROWS)
  int swap128_rows = 1024;  // auto: 128-token swap-AB tiles (fused GEMMs) up to this mean (MOE_GEMM_SWAP128_ROWS)
  int gemm_T = 0;        // tokens of the forward whose GEMMs are being enqueued
  // programmatic dependent launch of the small kernels (MOE_PDL_FRONT bit mask):
  // 1 block prefix + dispatch (eager), 2 combine (eager), 4 / 8 the same in CUDA graphs
  int pdl_front = 1;
  bool capturing = false;  // enqueue_forward is recording a CUDA graph
  bool pdl_prefix() const { return (pdl_front & (capturing ? 4 : 1)) != 0; }
  bool pdl_combine() const { return (pdl_front & (capturing ? 8 : 2)) != 0; }
  bool swap_fuse = true;
  // swap-AB GEMM2 in 128-row weight tiles (MOE_SWAP_HALF2=1; default 256 rows: the half tiles
  // re-read each tile's H rows and cost cfg5 +8 us, profiles/ab_frontend_r02.md)
  bool swap_half2 = false;  // swap-AB: GEMM1 and GEMM2 in one launch (MOE_SWAP_FUSE=0: two)
  // single GPU, <= 32 token blocks: gate, top-k, plan and dispatch in ONE cooperative launch
  // (kernels/frontend.cu; MOE_FRONTEND=0: the gate / finish / dispatch launches)
  bool frontend = true;
  // decode weight prefetch with the fused front end (MOE_FRONT_PREFETCH): the side-stream
  // kernel (default), or "inline": the front end's CTAs issue the bulk prefetches themselves
  bool front_prefetch_inline = false;
  bool trace_marker = false;  // MOE_FRONT_TRACE=2: + a marker kernel at the layer's start
  DevBuf<unsigned long long> front_trace;  // MOE_FRONT_TRACE=1: phase stamps of the fused front end (moe_buffer 12)
  bool fuse_plan = true;  // single GPU, <= 32 blocks: dispatch builds prefix + plan (MOE_FUSE_PLAN=0: block-prefix launch)
  // decode (swap-AB K4): MB of the first experts' weights prefetched into L2 on a side
  // stream while the front end runs (MOE_DECODE_PREFETCH_MB, default 64; 0 = off)
  int prefetch_mb = 64;
  cudaStream_t pstream = nullptr;
  cudaEvent_t ev_pf_fork = nullptr, ev_pf_join = nullptr, ev_front = nullptr;
  DevBuf<int> swap_ready; // its per-(segment, m-tile) GEMM1-done counters (+ CTA counter)
  int pred_distance = 1;  // predictor slot 0 scores layer + pred_distance
  int count_stride = 0;   // ints per rank in the counts buffer: E * (1 + n_pred)
  bool fp32 = false;      // MOE_PRECISION_FP32: SIMT fp32 path (K7)
  int elem = 1;           // 16-bit units per element (2 in fp32 mode)
  int xw = 0;             // one activation row in 16-bit units (d_model * elem)
  DevBuf<float> gu_f32;   // fp32 GEMM1 output [rows_cap][2 ff]
  DevBuf<float> gate_partial;  // split-K gate scratch (small batches)
  bool use_graphs = false;     // replay single-GPU forwards as CUDA graphs
  // K4 tile scheduler (MOE_GEMM_SCHED): 0 auto = the 2-SM kernel claims tiles from a global
  // counter (-24% DRAM bytes at cfg2, profiles/ab_2sm_sched_r02.md), the 1-SM kernel walks
  // them statically; 1 static everywhere; 2 dynamic everywhere (1-SM A/B: no gain)
  int sched_mode = 0;
  bool sched_2sm() const { return sched_mode != 1; }
  bool sched_1sm() const { return sched_mode == 2; }
  bool use_pdl = true;         // K4 launched programmatically behind its producer (MOE_PDL=0: off)
  // single GPU: GEMM1 gathers its A rows from x with TMA gather4 and the
  // dispatch kernel only ranks (MOE_GATHER=1).  Opt-in: bit-identical, but 32
  // gather4 instructions per 16 KB A stage make GEMM1 2.7x slower than one
  // tile load (profiles/ab_gather4_r01.md), far more than the copy it saves.
  bool gather = false;
  // single GPU: the combine runs in GEMM2's epilogue (MOE_FUSED_COMBINE=1).  Opt-in:
  // bit-identical, but no faster under the power cap at cfg2 and slower for
  // short-K shapes (the late rows' sums serialise on 4 epilogue warps),
  // profiles/ab_fused_combine_r01.md
  bool fuse_combine = false;
  bool fuse_y = true;  // 2-SM GEMM2 writes y directly at top-2 on one GPU (MOE_FUSED_Y=0: yp + combine kernel)
  bool skip_combine = false;  // MOE_DEBUG_SKIP_COMBINE=1: timing experiments only (y is not written)
  DevBuf<unsigned> gate_ticket;  // CTAs of the gate grid done (histogram mirror, self-resetting)
  DevBuf<int32_t> row_owner;  // [rows_cap] row -> t * k + j
  DevBuf<int32_t> comb_cnt;   // [Tmax * d / 256] arrivals per (token, GEMM2 n tile)
  int group_m[2] = {0, 0};  // K4 m-tiles per n sweep (0: the kernel's default; MOE_GEMM_GROUP_M=g1,g2)
  DevBuf<int32_t> perm_src;    // gathered GEMM1: permuted row -> token
  CUtensorMap tmX;             // gather4 map over the current x ({64, 1} box)
  CUtensorMap tmGate;          // the streaming gate's map over the current x ({64, 32} boxes)
  CUtensorMap tmGateTc;        // the tcgen05 gate's map over the current x ({64, 128} boxes)
  const void* tmGateTc_ptr = nullptr;
  int tmGateTc_T = -1;
  const void* tmGate_ptr = nullptr;
  int tmGate_T = -1;
  const void* tmX_ptr = nullptr;
  int tmX_T = -1;
  DevBuf<int> gemm_sched;      // [GEMM1 next, done, GEMM2 next, done], zero between launches
  std::map<GraphKey, cudaGraphExec_t> graphs;
  bool user_capture = false;                // between moe_graph_begin and moe_graph_end
  std::vector<cudaGraphExec_t> user_graphs;  // moe_graph_end's graphs (id = index)
  // K4 timing ring: events around GEMM1 / GEMM2 of every forward (no sync)
  static constexpr int kGemmRing = 64;
  cudaEvent_t gemm_ev[kGemmRing][3] = {};
  int64_t gemm_rows[kGemmRing] = {};
  int64_t gemm_seq = 0;
  cudaStream_t stream = nullptr;
  ncclComm_t comm = nullptr;
  std::unique_ptr<Transport> transport;  // chunked exchange (NCCL / COPY); null for P2P and EXTERNAL
  std::vector<Layer> layers;
  // workspace
  DevBuf<int32_t> ids, counts, counts_all, block_counts, block_pre, pred_counts;
  DevBuf<float> wts;
  DevBuf<uint32_t> row_code;
  DevBuf<uint16_t> xp, h, yp, send, ret, x_in, y_out;
  // pipelined host-buffer forward: two slots of staging buffers + events
  cudaStream_t h2d = nullptr, d2h = nullptr;
  DevBuf<uint16_t> xa[2], ya[2];
  cudaEvent_t ev_x_ready[2] = {}, ev_x_free[2] = {}, ev_y_ready[2] = {}, ev_done[2] = {};
  static constexpr int kTicketRing = 16;
  cudaEvent_t ev_ticket[kTicketRing] = {};  // per-call completion (result in host memory)
  int64_t next_ticket = 0;
  DevBuf<DevPlan> dplan;
  int64_t rows_cap = 0, send_cap = 0;
  CUtensorMap tmA1, tmA2;    // 128-row boxes
  CUtensorMap tmA1w, tmA2w;  // 256-row boxes (256-row single-CTA K4 variant)
  CUtensorMap tmA1s, tmA2s;  // 32-row boxes (swap-AB decode variant: tokens are the N operand)
  // host staging (pinned)
  DevPlan* hplan = nullptr;
  int32_t* h_counts = nullptr;  // [G][E]
  uint16_t* wg_stage = nullptr;  // pinned staging for stream-ordered gate updates
  size_t wg_stage_bytes = 0;
  cudaEvent_t ev_wg_staged = nullptr;
  HostPlan plan;
  moeless::ReplicaRegistry registry{0};
  EventSet events;
  // staged-forward state
  int cur_layer = -1, cur_T = 0;
  const uint16_t* cur_x = nullptr;
  std::vector<int64_t> last_counts;
  int last_warm = 0, last_cold = 0;
  // single-GPU forward: host planner work deferred until the histogram lands
  PendingPlan pending;
  cudaEvent_t ev_counts = nullptr;
  // forwards on a caller stream: ordered against the ctx stream's uploads
  cudaEvent_t ev_ctx_tail = nullptr, ev_fwd_tail = nullptr;
  // caller-given routing (moe_layer_forward_ids): replaces K1 for one forward
  bool ext_route = false;
  const int32_t* ext_ids = nullptr;
  const float* ext_wts = nullptr;
  int* ids_err = nullptr;  // mapped pinned: 1 + first token with invalid ids (0 = none)
  // peer-memory exchange (MOE_EXCHANGE_P2P): one exported slab per rank
  bool p2p = false, p2p_ready = false;
  DevBuf<uint8_t> slab;
  size_t off_flags = 0, off_counts = 0, off_xp = 0, off_yp = 0;
  std::vector<void*> ipc_opened;  // peer slabs opened with cudaIpcOpenMemHandle
  PeerSlabs peers{};
  RowTargets xp_targets{}, yp_targets{};  // rank g -> g's xp / yp
  DevBuf<uint32_t> epoch_dev;              // the current forward's epoch (device; counts kernel increments)
  int* p2p_err = nullptr;                  // mapped pinned: first timed-out wait (1 + kind*8 + rank)
  DevBuf<uint32_t> dispatch_counter;       // CTAs of the signalling dispatch grid that finished
  uint64_t p2p_timeout_ns = 10000000000ull;
  // expert weight residency (MOE_RESIDENCY_PLACED): per layer [home slots | cache
  // slots] of W13 then W2 inside the slab, so peers can copy home experts out
  bool placed = false;
  int home_slots = 0, cache_slots = 0, slots = 0;
  size_t off_weights = 0, layer_wbytes = 0, w13_slot_bytes = 0, w2_slot_bytes = 0;
  uint8_t* peer_base[kMaxRanks] = {};
  cudaStream_t wstream = nullptr;        // weight copies (copy engines, off the compute stream)
  cudaEvent_t ev_peers_ready = nullptr;  // after the first forward's cross-rank handshake
  bool peers_ready = false;
};

// helpers shared between the context and the forward translation units
namespace moe {
Layer& layer_at(moe_ctx* c, int layer);
void ensure_pools(moe_ctx* c, Layer& L);
void ensure_placement(moe_ctx* c, int layer);
void plan_layer(moe_ctx* c, int layer, const std::vector<int64_t>& loads, long iteration);
void issue_weight_copies(moe_ctx* c, int layer);
void flush_pending_plan(moe_ctx* c);
}  // namespace moe
