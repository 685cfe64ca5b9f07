// capi.cpp — the C-ABI drop-in boundary (include/moe_b200.h).
//
// Owns one device's share of the MoE layer: weight pools (and, with
// MOE_RESIDENCY_PLACED, the replica weight slots), workspace, TMA descriptors,
// streams, the peer-memory slab or NCCL communicator, and sequences a layer
// forward (enqueue_forward):
//
//   K1 gate + top-k + histogram (+K2 predictor)        gate.cu
//   G > 1: counts exchange (peer slabs, or NCCL all-gather)
//   plan: on the device (G = 1, or placement planned ahead) or on the host
//         (scale_experts / place_experts on the actual loads, exchange plan)
//   block prefix + K3 dispatch (peer stores at G > 1)  dispatch.cu
//   K4 GEMM1 (SwiGLU) + GEMM2                          ffn_gemm.cu  (tcgen05/TMEM/TMA)
//   K5 combine (peer loads at G > 1)                   dispatch.cu
//
// Replaces layer_forward_time (proj/src/cost_model.cpp:91-122) for callers
// that want the real layer instead of the analytic model.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
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

#include "host/exchange_plan.h"
#include "kernels/dispatch_plan.h"
#include "moe_b200.h"
#include "moeless/api.hpp"

namespace moe {
// kernels
int gate_num_blocks(int T);
cudaError_t launch_gate_topk(const __nv_bfloat16* x, int T, int d, const __nv_bfloat16* w_all, int E, int n_pred,
                             int k, int32_t* ids, float* wts, int32_t* counts, int32_t* block_counts,
                             int32_t* pred_counts, float* partial, cudaStream_t stream);
cudaError_t launch_block_prefix(const int32_t* block_counts, int nblk, int E, const DevPlan* plan,
                                int32_t* block_pre, cudaStream_t s);
cudaError_t launch_dispatch(const __nv_bfloat16* x, int T, int d, int E, int k, const int32_t* ids,
                            const int32_t* block_pre, const DevPlan* plan, const RowTargets& targets,
                            uint32_t* row_code, const PeerSignal& sig, cudaStream_t s, int32_t* perm_src,
                            int32_t* row_owner);
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
cudaError_t launch_plan_local(const int32_t* counts, int E, DevPlan* plan, cudaStream_t s);
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
                           const float* wts, __nv_bfloat16* y, int num_sms, cudaStream_t s);
cudaError_t launch_grouped_gemm_m256(int epi, const CUtensorMap* tmA, const CUtensorMap* tmB, const GemmSeg* segs,
                                     const int* nseg, int n_total, int k_total, int b_rows_per_slot,
                                     __nv_bfloat16* out, int out_ld, int num_ctas, cudaStream_t stream);
cudaError_t launch_grouped_gemm_2sm(int epi, const CUtensorMap* tmA, const CUtensorMap* tmB, const GemmSeg* segs,
                                    const int* nseg, int n_total, int k_total, int b_rows_per_slot,
                                    __nv_bfloat16* out, int out_ld, int num_ctas, cudaStream_t stream);
cudaError_t launch_grouped_gemm(int epi, const CUtensorMap* tmA, const CUtensorMap* tmB, const GemmSeg* segs,
                                const int* nseg, int n_total, int k_total, int b_rows_per_slot,
                                __nv_bfloat16* out, int out_ld, int num_ctas, cudaStream_t stream, int* sched,
                                bool pdl, const int32_t* a_gather, int group_m, const FusedCombine& fc);
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
namespace {
thread_local std::string g_last_error;

struct Status : std::runtime_error {
  int code;
  Status(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CU_CHECK(expr)                                                                      \
  do {                                                                                      \
    cudaError_t _e = (expr);                                                                \
    if (_e != cudaSuccess)                                                                  \
      throw Status(MOE_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));          \
  } while (0)

template <class F>
int guarded(F&& f) {
  try {
    f();
    return MOE_OK;
  } catch (const Status& s) {
    g_last_error = s.what();
    return s.code;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return MOE_EINVAL;
  } catch (const std::runtime_error& e) {
    g_last_error = e.what();
    return MOE_EINFEASIBLE;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return MOE_ESTATE;
  }
}

constexpr size_t pad16(size_t b) { return (b + 15) & ~size_t(15); }
static_assert(sizeof(DevPlan) % 16 == 0, "DevPlan is copied in 16-byte words");
static_assert(sizeof(PlacementTable) % 16 == 0, "PlacementTable is copied in 16-byte words");

void require(bool ok, const std::string& msg) {
  if (!ok) throw std::invalid_argument(msg);
}

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
NcclApi g_nccl;

// ================================================================ TMA maps
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
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
CUtensorMap make_kmajor_map(const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
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
  // layer-aware predictor state (MOE_PLAN_PREDICTED)
  std::vector<int64_t> pred_loads;          // predicted loads for this layer (made d layers earlier)
  bool pred_valid = false;
  long plan_for = -1;                       // iteration whose placement was planned ahead
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
  bool operator<(const GraphKey& o) const {
    return std::tie(layer, T, x, y, x_consumed, pred) < std::tie(o.layer, o.T, o.x, o.y, o.x_consumed, o.pred);
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

}  // namespace

// =================================================================== context
struct moe_ctx {
  moe_ctx_desc desc{};
  int E = 0, k = 0, d = 0, ff = 0, G = 1, rank = 0, Tmax = 0, n_pred = 0, num_sms = 148;
  int gemm_variant = 0;  // 0 auto, 1 force 1-SM, 2 force 2-SM (env MOE_GEMM_VARIANT=1sm|2sm)
  int pred_distance = 1;  // predictor slot 0 scores layer + pred_distance
  int count_stride = 0;   // ints per rank in the counts buffer: E * (1 + n_pred)
  bool fp32 = false;      // MOE_PRECISION_FP32: SIMT fp32 path (K7)
  int elem = 1;           // 16-bit units per element (2 in fp32 mode)
  int xw = 0;             // one activation row in 16-bit units (d_model * elem)
  DevBuf<float> gu_f32;   // fp32 GEMM1 output [rows_cap][2 ff]
  DevBuf<float> gate_partial;  // split-K gate scratch (small batches)
  bool use_graphs = false;     // replay single-GPU forwards as CUDA graphs
  bool dyn_sched = false;      // K4 claims tiles from a global counter (MOE_GEMM_SCHED=dynamic; A/B: no gain)
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
  DevBuf<int32_t> row_owner;  // [rows_cap] row -> t * k + j
  DevBuf<int32_t> comb_cnt;   // [Tmax * d / 256] arrivals per (token, GEMM2 n tile)
  int group_m[2] = {0, 0};  // K4 m-tiles per n sweep (0: the kernel's default; MOE_GEMM_GROUP_M=g1,g2)
  DevBuf<int32_t> perm_src;    // gathered GEMM1: permuted row -> token
  CUtensorMap tmX;             // gather4 map over the current x ({64, 1} box)
  const void* tmX_ptr = nullptr;
  int tmX_T = -1;
  DevBuf<int> gemm_sched;      // [GEMM1 next, done, GEMM2 next, done], zero between launches
  std::map<GraphKey, cudaGraphExec_t> graphs;
  // K4 timing ring: events around GEMM1 / GEMM2 of every forward (no sync)
  static constexpr int kGemmRing = 64;
  cudaEvent_t gemm_ev[kGemmRing][3] = {};
  int64_t gemm_rows[kGemmRing] = {};
  int64_t gemm_seq = 0;
  cudaStream_t stream = nullptr;
  ncclComm_t comm = nullptr;
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

namespace {

void stage_gate(moe_ctx* c, Layer& L, const uint16_t* x, int T, cudaStream_t s, int32_t* pred_counts) {
  require(L.has_gate, "gate weights not set for layer");
  CU_CHECK(cudaMemsetAsync(c->counts.p, 0, sizeof(int32_t) * c->count_stride, s));
  if (c->fp32) {
    CU_CHECK(launch_gate_f32(reinterpret_cast<const float*>(x), T, c->d, reinterpret_cast<const float*>(L.wg.p), c->E,
                             c->k, c->ids.p, c->wts.p, c->counts.p, c->block_counts.p, s));
    return;
  }
  CU_CHECK(launch_gate_topk(reinterpret_cast<const __nv_bfloat16*>(x), T, c->d,
                            reinterpret_cast<const __nv_bfloat16*>(L.wg.p), c->E, pred_counts ? c->n_pred : 0,
                            c->k, c->ids.p, c->wts.p, c->counts.p, c->block_counts.p,
                            pred_counts ? pred_counts : c->pred_counts.p, c->gate_partial.p, s));
}

void ensure_pools(moe_ctx* c, Layer& L);

// MOE_RESIDENCY_PLACED: issue the layer's pending weight copies on the weight
// stream — each cold expert's W13/W2 from its home rank's slot (peer memory
// over NVLink, copy engines) into the cache slot chosen for it.  The stream
// first waits for the layer's last enqueued GEMMs (the slot may hold an
// evicted expert they still read); the layer's next GEMM1 waits for ev_wready.
// Before the first forward's cross-rank handshake a peer may not have loaded
// its home experts yet, so copies wait for it (issued from enqueue_forward).
void issue_weight_copies(moe_ctx* c, int layer) {
  Layer& L = c->layers[layer];
  if (L.pending_copies.empty() || !c->peers_ready) return;
  if (L.used_recorded) CU_CHECK(cudaStreamWaitEvent(c->wstream, L.ev_used, 0));
  CU_CHECK(cudaEventRecord(L.ev_wstart, c->wstream));
  const size_t lo = static_cast<size_t>(layer) * c->layer_wbytes;
  const size_t w2_base = static_cast<size_t>(c->slots) * c->w13_slot_bytes;
  uint8_t* dst = c->slab.p + c->off_weights + lo;
  for (const auto& sc : L.pending_copies) {
    const int slot = sc.first, e = sc.second;
    const uint8_t* src = c->peer_base[e % c->G] + c->off_weights + lo;
    const size_t hs = static_cast<size_t>(e / c->G);
    CU_CHECK(cudaMemcpyAsync(dst + slot * c->w13_slot_bytes, src + hs * c->w13_slot_bytes, c->w13_slot_bytes,
                             cudaMemcpyDefault, c->wstream));
    CU_CHECK(cudaMemcpyAsync(dst + w2_base + slot * c->w2_slot_bytes, src + w2_base + hs * c->w2_slot_bytes,
                             c->w2_slot_bytes, cudaMemcpyDefault, c->wstream));
  }
  CU_CHECK(cudaEventRecord(L.ev_wready, c->wstream));
  L.wready_valid = true;
  L.wready_timed = true;
  L.pending_copies.clear();
}

// MOE_RESIDENCY_PLACED: make every expert that has a replica on this rank
// resident — its home slot, the cache slot it already occupies (warm: the
// ReplicaRegistry keep-alive made physical, placer.cpp:84-92), or a free /
// least-recently-used cache slot it is copied into (cold).  Co-located
// replicas of one expert share one slot (they are one GEMM segment).
void apply_residency(moe_ctx* c, int layer) {
  Layer& L = c->layers[layer];
  if (!c->placed) return;
  ensure_pools(c, L);
  const long stamp = L.placements + 1;
  std::vector<char> need(c->E, 0);
  size_t f = 0;
  for (int e = 0; e < c->E; ++e)
    for (int r = 0; r < L.rep_counts[e]; ++r, ++f)
      if (L.rep_gpu[f] == c->rank) need[e] = 1;
  // decide on copies of the slot state; the layer keeps its residency if the
  // placement does not fit
  std::vector<int> slot_of = L.slot_of, cache_expert = L.cache_expert;
  std::vector<long> cache_stamp = L.cache_stamp;
  std::vector<std::pair<int, int>> fills;
  int hits = 0;
  for (int e = 0; e < c->E; ++e)
    if (need[e] && e % c->G != c->rank && slot_of[e] >= 0) {
      cache_stamp[slot_of[e] - c->home_slots] = stamp;
      ++hits;
    }
  for (int e = 0; e < c->E; ++e) {
    if (!need[e] || e % c->G == c->rank || slot_of[e] >= 0) continue;
    int best = -1;  // a free slot (stamp -1) or the least recently needed one this placement does not use
    for (int i = 0; i < c->cache_slots; ++i) {
      const int ce = cache_expert[i];
      if (ce >= 0 && need[ce]) continue;
      if (best < 0 || cache_stamp[i] < cache_stamp[best]) best = i;
    }
    if (best < 0)
      throw Status(MOE_EINFEASIBLE, "no replica slot free for expert " + std::to_string(e) + " of layer " +
                                        std::to_string(layer) + " on GPU " + std::to_string(c->rank) + " (" +
                                        std::to_string(c->cache_slots) + " cache slots)");
    if (cache_expert[best] >= 0) slot_of[cache_expert[best]] = -1;  // evicted
    cache_expert[best] = e;
    cache_stamp[best] = stamp;
    slot_of[e] = c->home_slots + best;
    fills.emplace_back(c->home_slots + best, e);
  }
  const int copies = static_cast<int>(fills.size());
  L.placements = stamp;
  L.slot_of.swap(slot_of);
  L.cache_expert.swap(cache_expert);
  L.cache_stamp.swap(cache_stamp);
  L.pending_copies.insert(L.pending_copies.end(), fills.begin(), fills.end());
  L.copies_last = copies;
  L.hits_last = hits;
  if (copies == 0) L.wready_timed = false;
  issue_weight_copies(c, layer);
}

// The placement changed (planner, moe_set_placement or default): make its
// replicas resident (PLACED) and refresh the device copy the on-device
// exchange planner reads (peer-memory contexts).
void placement_changed(moe_ctx* c, int layer) {
  Layer& L = c->layers[layer];
  L.has_placement = true;
  if (!c->p2p) return;
  apply_residency(c, layer);
  const int R = static_cast<int>(L.rep_gpu.size());
  if (R > kMaxReplicas) throw std::invalid_argument("too many replicas in one layer");
  if (!L.ptab.p) {
    L.ptab.alloc(1);
    CU_CHECK(cudaHostAlloc(&L.h_ptab, sizeof(PlacementTable), cudaHostAllocMapped));
    CU_CHECK(cudaEventCreateWithFlags(&L.ev_ptab, cudaEventDisableTiming));
  } else {
    CU_CHECK(cudaEventSynchronize(L.ev_ptab));  // the previous upload has left the staging copy
  }
  PlacementTable& t = *L.h_ptab;
  t.E = c->E;
  t.R = R;
  int f = 0;
  for (int e = 0; e < c->E; ++e) {
    t.rep_base[e] = f;
    for (int r = 0; r < L.rep_counts[e]; ++r, ++f) t.expert_of[f] = e;
  }
  t.rep_base[c->E] = f;
  for (int i = 0; i < R; ++i) t.gpu_of[i] = L.rep_gpu[i];
  for (int e = 0; e < c->E; ++e) t.slot_of[e] = c->placed ? std::max(0, L.slot_of[e]) : e;
  // SM copy from mapped memory: never queues behind bulk token copies
  CU_CHECK(launch_small_copy(L.ptab.p, L.h_ptab, sizeof(PlacementTable), c->stream));
  CU_CHECK(cudaEventRecord(L.ev_ptab, c->stream));
}

// default: one replica per expert, expert e on GPU e mod G (static_plan, baselines.cpp:32-60)
void ensure_placement(moe_ctx* c, int layer) {
  Layer& L = c->layers[layer];
  if (L.has_placement) return;
  L.rep_counts.assign(c->E, 1);
  L.rep_gpu.resize(c->E);
  for (int e = 0; e < c->E; ++e) L.rep_gpu[e] = e % c->G;
  placement_changed(c, layer);
}

// Decide the placement for this forward (host), then build + upload the plan.
// MoEless planning for one layer on a load vector: scale_experts (Alg. 1) ->
// place_experts (Alg. 2) against the keep-alive registry -> update_registry
// (the reference's per-layer sequence, simulator.cpp:159-201).
void plan_layer(moe_ctx* c, int layer, const std::vector<int64_t>& loads, long iteration) {
  Layer& L = c->layers[layer];
  moeless::ModelSpec ms;
  ms.num_layers = std::max(1, c->desc.num_layers);
  ms.experts_per_layer = c->E;
  ms.top_k = c->k;
  ms.expert_mem_mb = c->desc.expert_mem_mb > 0 ? c->desc.expert_mem_mb : 3.0 * c->d * c->ff * 2 / 1e6;
  ms.layer_mem_cap_mb = c->desc.layer_mem_cap_mb;
  moeless::ScalerConfig sc;
  sc.cv_threshold = c->desc.cv_threshold;
  auto sp = moeless::scale_experts(moeless::LoadVector{layer, loads}, ms, sc);
  moeless::ClusterSpec cl;
  cl.gpu_count = c->G;
  cl.gpu_mem_capacity_mb = c->desc.gpu_mem_capacity_mb > 0 ? c->desc.gpu_mem_capacity_mb : 180000.0;
  auto pr = moeless::place_experts(sp, cl, c->registry, iteration);
  moeless::update_registry(c->registry, pr.placement, iteration);
  L.warm = pr.warm_count;
  L.cold = pr.cold_count;
  L.rep_counts.assign(sp.replica_counts.begin(), sp.replica_counts.end());
  L.rep_gpu.clear();
  for (auto& v : pr.placement.gpu_for) L.rep_gpu.insert(L.rep_gpu.end(), v.begin(), v.end());
  placement_changed(c, layer);
}

// buf: [G][stride] int32 from the gate — per rank, E actual counts followed by
// n_pred x E predictor counts (stride == E when no predictor ran).
void stage_plan(moe_ctx* c, int layer, int plan_mode, long iteration, const int32_t* buf, int stride) {
  Layer& L = c->layers[layer];
  std::vector<int64_t> all(static_cast<size_t>(c->G) * c->E);
  std::vector<int64_t> total(c->E, 0), predicted(c->E, 0);
  const bool have_pred = stride >= 2 * c->E;
  for (int s = 0; s < c->G; ++s)
    for (int e = 0; e < c->E; ++e) {
      all[static_cast<size_t>(s) * c->E + e] = buf[static_cast<size_t>(s) * stride + e];
      total[e] += buf[static_cast<size_t>(s) * stride + e];
      if (have_pred) predicted[e] += buf[static_cast<size_t>(s) * stride + c->E + e];
    }
  c->last_counts = total;
  // realised accuracy of the prediction made d layers earlier (predictor.cpp:168-186)
  L.last_accuracy = -1.0;
  if (L.pred_valid) {
    L.last_accuracy = moeless::measure_accuracy({layer, L.pred_loads}, {layer, total});
    L.acc_sum += L.last_accuracy;
    ++L.acc_n;
    L.pred_valid = false;
  }
  if (plan_mode == MOE_PLAN_SYNC) {
    // synchronous planning on the actual loads (oracle predictor, distance 0)
    plan_layer(c, layer, total, iteration);
    L.plan_source = 1;
  } else if (plan_mode == MOE_PLAN_PREDICTED && L.plan_for != iteration) {
    // no prediction reached this layer (l < d, simulator.cpp:146-151): bootstrap
    // from the layer's load history with the historical predictor
    moeless::PredictorProfile hp;
    hp.kind = moeless::PredictorKind::historical;
    const auto guess = moeless::predict({layer, total}, L.history, hp, iteration, 1);
    plan_layer(c, layer, guess.loads, iteration);
    L.plan_source = 3;
    ++L.bootstraps;
  } else if (plan_mode == MOE_PLAN_PREDICTED) {
    L.plan_source = 2;  // placement made d layers ago from the predictor
  } else {
    ensure_placement(c, layer);
  }
  // plan layer + d from this layer's predictor histogram (the MoEless
  // layer-aware predictor: plan ahead, evaluate on the actual loads)
  const int target = layer + c->pred_distance;
  if (have_pred && target < static_cast<int>(c->layers.size())) {
    Layer& Lt = c->layers[target];
    Lt.pred_loads = predicted;
    Lt.pred_valid = true;
    if (plan_mode == MOE_PLAN_PREDICTED) {
      plan_layer(c, target, predicted, iteration);
      Lt.plan_for = iteration;
    }
  }
  L.history.push_back({layer, total});
  if (L.history.size() > 16) L.history.erase(L.history.begin());
  build_exchange_plan(c->G, c->rank, c->E, all.data(), L.rep_counts.data(), L.rep_gpu.data(), c->plan, c->p2p);
  if (c->placed)  // GEMM segments read the expert's resident slot, not the expert index
    for (int i = 0; i < c->plan.dev.nseg; ++i) {
      GemmSeg& g = c->plan.dev.segs[i];
      require(L.slot_of[g.slot] >= 0, "expert " + std::to_string(g.slot) + " has rows here but is not resident");
      g.slot = L.slot_of[g.slot];
    }
  if (c->plan.rows_local > c->rows_cap || (!c->p2p && c->plan.rows_send > c->send_cap))
    throw Status(MOE_EINFEASIBLE, "received rows exceed workspace capacity");
  *c->hplan = c->plan.dev;
}

void stage_dispatch(moe_ctx* c, const uint16_t* x, int T, cudaStream_t s, bool upload_plan = true,
                    bool gather = false, bool fused = false) {
  if (upload_plan)
    CU_CHECK(launch_small_copy(c->dplan.p, c->hplan, sizeof(DevPlan), s));  // SM copy from mapped pinned memory
  const int nblk = gate_num_blocks(T);
  CU_CHECK(launch_block_prefix(c->block_counts.p, nblk, c->E, c->dplan.p, c->block_pre.p, s));
  // rows move as opaque 16-byte chunks: the row width in 16-bit units covers fp32 rows too
  RowTargets t{};
  PeerSignal sig{};
  if (c->p2p) {
    t = c->xp_targets;  // rows go straight into the owning rank's received-rows buffer
    if (T > 0) {        // the dispatch grid itself publishes "my rows are delivered"
      for (int g = 0; g < c->G; ++g) sig.flags[g] = c->peers.flags[g];
      sig.counter = c->dispatch_counter.p;
      sig.G = c->G;
      sig.src = c->rank;
      sig.kind = kFlagRows;
      sig.epoch = c->epoch_dev.p;
    }
  } else {
    t.base[0] = c->xp.p;
    t.base[kSendTarget] = c->send.p;
  }
  CU_CHECK(launch_dispatch(reinterpret_cast<const __nv_bfloat16*>(x), T, c->xw, c->E, c->k, c->ids.p, c->block_pre.p,
                           c->dplan.p, t, c->row_code.p, sig, s, gather ? c->perm_src.p : nullptr,
                           fused ? c->row_owner.p : nullptr));
}

// The exchange step of one direction.  NCCL: grouped send/recv, forward: my
// send buffer -> peers' received-rows buffers; backward: my Y rows -> peers'
// return buffers.  Peer memory: the rows already moved inside dispatch (and
// combine reads peers' outputs in place), so only the flag handshake is left:
// forward = "my rows are in your buffer", backward = "my outputs are ready".
void stage_exchange(moe_ctx* c, bool forward, cudaStream_t s) {
  if (c->G == 1) return;
  if (c->p2p) {
    const int kind = forward ? kFlagRows : kFlagOutputs;
    // the rows signal is fused into the dispatch kernel (a rank without tokens
    // launches no dispatch and signals here)
    if (!forward || c->cur_T == 0)
      CU_CHECK(launch_p2p_signal(c->peers, c->G, kind, c->rank, c->epoch_dev.p, s));
    CU_CHECK(launch_p2p_wait(c->peers.flags[c->rank], c->G, kind, c->epoch_dev.p, c->p2p_timeout_ns, c->p2p_err, s));
    return;
  }
  if (c->desc.exchange_mode != MOE_EXCHANGE_NCCL) return;
  const size_t w = static_cast<size_t>(c->xw);  // row width in 16-bit units (bf16 or fp32 rows)
  const size_t row_bytes = w * 2;
  g_nccl.check(g_nccl.GroupStart(), "ncclGroupStart");
  if (forward) {
    for (const Chunk& ch : c->plan.sends)
      g_nccl.check(g_nccl.Send(c->send.p + ch.row_offset * w, ch.rows * row_bytes, ncclUint8, ch.peer, c->comm, s),
                   "ncclSend");
    for (const Chunk& ch : c->plan.recvs)
      g_nccl.check(g_nccl.Recv(c->xp.p + ch.row_offset * w, ch.rows * row_bytes, ncclUint8, ch.peer, c->comm, s),
                   "ncclRecv");
  } else {
    for (const Chunk& ch : c->plan.recvs)
      g_nccl.check(g_nccl.Send(c->yp.p + ch.row_offset * w, ch.rows * row_bytes, ncclUint8, ch.peer, c->comm, s),
                   "ncclSend");
    for (const Chunk& ch : c->plan.sends)
      g_nccl.check(g_nccl.Recv(c->ret.p + ch.row_offset * w, ch.rows * row_bytes, ncclUint8, ch.peer, c->comm, s),
                   "ncclRecv");
  }
  g_nccl.check(g_nccl.GroupEnd(), "ncclGroupEnd");
}

// K4: which = 0 -> GEMM1 (X -> H, SwiGLU epilogue), 1 -> GEMM2 (H -> Y).
// Default: the 1-SM kernel.  The 2-SM (cta_group::2, 256-row tile) kernel
// reaches ~88% tensor-pipe utilisation per clock vs ~80%, but under the
// B200's 1 kW cap it settles ~190 MHz lower and nets ~4% less throughput on
// the Mixtral layer (profiles/ab_gemm_variants_r01.md), so it is opt-in
// (MOE_GEMM_VARIANT=2sm) until it is made more energy-efficient.
void launch_ffn_gemm(moe_ctx* c, int layer, int which, cudaStream_t s, int64_t rows = 0, bool gather = false,
                     uint16_t* fused_y = nullptr) {
  Layer& L = c->layers[layer];
  if (c->fp32) {  // K7: SIMT fp32 grouped GEMMs (+ SwiGLU pass between them)
    const GemmSeg* segs = c->dplan.p->segs;
    const int* nseg = &c->dplan.p->nseg;
    if (which == 0) {
      CU_CHECK(launch_grouped_sgemm(reinterpret_cast<const float*>(c->xp.p), c->d,
                                    reinterpret_cast<const float*>(L.w13.p), 2 * c->ff, c->d, segs, nseg, 2 * c->ff,
                                    c->d, c->gu_f32.p, 2 * c->ff, c->num_sms, s));
      CU_CHECK(launch_swiglu_f32(c->gu_f32.p, static_cast<int>(rows), c->ff, reinterpret_cast<float*>(c->h.p), s));
    } else {
      CU_CHECK(launch_grouped_sgemm(reinterpret_cast<const float*>(c->h.p), c->ff,
                                    reinterpret_cast<const float*>(L.w2.p), c->d, c->ff, segs, nseg, c->d, c->ff,
                                    reinterpret_cast<float*>(c->yp.p), c->d, c->num_sms, s));
    }
    return;
  }
  const bool two_sm = c->gemm_variant == 2, m256 = c->gemm_variant == 3;
  if (two_sm || m256) {
    auto fn = two_sm ? launch_grouped_gemm_2sm : launch_grouped_gemm_m256;
    const CUtensorMap* a1 = m256 ? &c->tmA1w : &c->tmA1;
    const CUtensorMap* a2 = m256 ? &c->tmA2w : &c->tmA2;
    if (which == 0)
      CU_CHECK(fn(0, a1, two_sm ? &L.tmB1h : &L.tmB1, c->dplan.p->segs, &c->dplan.p->nseg, 2 * c->ff, c->d,
                  2 * c->ff, reinterpret_cast<__nv_bfloat16*>(c->h.p), c->ff, c->num_sms, s));
    else
      CU_CHECK(fn(1, a2, two_sm ? &L.tmB2h : &L.tmB2, c->dplan.p->segs, &c->dplan.p->nseg, c->d, c->ff, c->d,
                  reinterpret_cast<__nv_bfloat16*>(c->yp.p), c->d, c->num_sms, s));
    return;
  }
  // 1-SM kernel with the dynamic tile scheduler (counter pair per GEMM)
  int* sched = c->dyn_sched ? c->gemm_sched.p + 2 * which : nullptr;
  if (which == 0)
    CU_CHECK(launch_grouped_gemm(0, gather ? &c->tmX : &c->tmA1, &L.tmB1, c->dplan.p->segs, &c->dplan.p->nseg,
                                 2 * c->ff, c->d, 2 * c->ff, reinterpret_cast<__nv_bfloat16*>(c->h.p), c->ff,
                                 c->num_sms, s, sched, c->use_pdl, gather ? c->perm_src.p : nullptr, c->group_m[0],
                                 FusedCombine{}));
  else {
    FusedCombine fc{};
    if (fused_y) {
      fc.row_owner = c->row_owner.p;
      fc.row_code = c->row_code.p;
      fc.wts = c->wts.p;
      fc.counters = c->comb_cnt.p;
      fc.y = fused_y;
      fc.k = c->k;
    }
    CU_CHECK(launch_grouped_gemm(1, &c->tmA2, &L.tmB2, c->dplan.p->segs, &c->dplan.p->nseg, c->d, c->ff, c->d,
                                 reinterpret_cast<__nv_bfloat16*>(c->yp.p), c->d, c->num_sms, s, sched, c->use_pdl,
                                 nullptr, c->group_m[1], fc));
  }
}

void stage_expert(moe_ctx* c, int layer, cudaStream_t s) {
  launch_ffn_gemm(c, layer, 0, s, c->plan.rows_local);
  launch_ffn_gemm(c, layer, 1, s, c->plan.rows_local);
}

void stage_combine(moe_ctx* c, uint16_t* y, int T, cudaStream_t s) {
  RowTargets t{};
  if (c->p2p) {
    t = c->yp_targets;  // expert outputs are read where they were computed
  } else {
    t.base[0] = c->yp.p;
    t.base[kSendTarget] = c->ret.p;
  }
  if (c->fp32) {
    CU_CHECK(launch_combine_f32(t, T, c->d, c->k, c->row_code.p, c->wts.p, reinterpret_cast<float*>(y), s));
    return;
  }
  CU_CHECK(launch_combine(t, T, c->d, c->k, c->row_code.p, c->wts.p, reinterpret_cast<__nv_bfloat16*>(y),
                          c->num_sms, s));
}

void check_p2p(moe_ctx* c) {
  if (!c->p2p || !c->p2p_err || *reinterpret_cast<volatile int*>(c->p2p_err) == 0) return;
  const int v = *c->p2p_err - 1;
  static const char* kinds[] = {"gate counts", "dispatched rows", "expert outputs", "?"};
  throw Status(MOE_ESTATE, std::string("peer exchange timed out waiting for ") + kinds[(v / kMaxRanks) & 3] +
                               " of rank " + std::to_string(v % kMaxRanks) + " (ranks out of step?)");
}

cudaStream_t pick(moe_ctx* c, void* s) { return s ? static_cast<cudaStream_t>(s) : c->stream; }

// Run the host planner for the last single-GPU forward once its histogram is
// in mapped host memory (waits only for that forward's gate kernel).
void flush_pending_plan(moe_ctx* c) {
  if (!c->pending.active) return;
  c->pending.active = false;
  CU_CHECK(cudaEventSynchronize(c->ev_counts));
  check_p2p(c);
  stage_plan(c, c->pending.layer, c->pending.mode, c->pending.iteration, c->h_counts, c->pending.stride);
  if (c->pending.gemm_slot >= 0) c->gemm_rows[c->pending.gemm_slot] = c->plan.rows_local;
}

Layer& layer_at(moe_ctx* c, int layer) {
  require(c != nullptr, "null context");
  require(layer >= 0 && layer < static_cast<int>(c->layers.size()), "layer out of range");
  return c->layers[layer];
}

void ensure_pools(moe_ctx* c, Layer& L) {
  if (L.w13.p) return;
  // weight slots: one per expert (ALL), or home + cache slots inside the slab (PLACED)
  const int nslots = c->placed ? c->slots : c->E;
  if (c->placed) {
    const size_t li = static_cast<size_t>(&L - c->layers.data());
    uint8_t* base = c->slab.p + c->off_weights + li * c->layer_wbytes;
    L.w13.view(base, static_cast<size_t>(nslots) * 2 * c->ff * c->d);
    L.w2.view(base + static_cast<size_t>(nslots) * c->w13_slot_bytes, static_cast<size_t>(nslots) * c->d * c->ff);
    L.slot_of.assign(c->E, -1);
    for (int e = c->rank; e < c->E; e += c->G) L.slot_of[e] = e / c->G;  // home experts
    L.cache_expert.assign(c->cache_slots, -1);
    L.cache_stamp.assign(c->cache_slots, -1);
    CU_CHECK(cudaEventCreateWithFlags(&L.ev_used, cudaEventDisableTiming));
    CU_CHECK(cudaEventCreate(&L.ev_wstart));
    CU_CHECK(cudaEventCreate(&L.ev_wready));
  } else {
    L.w13.alloc(static_cast<size_t>(nslots) * 2 * c->ff * c->d * c->elem);
    L.w2.alloc(static_cast<size_t>(nslots) * c->d * c->ff * c->elem);
  }
  L.expert_loaded.assign(c->E, 0);
  if (c->fp32) return;  // SIMT fp32 path: no tensor maps
  L.tmB1 = make_kmajor_map(L.w13.p, static_cast<uint64_t>(nslots) * 2 * c->ff, c->d, 256);
  L.tmB2 = make_kmajor_map(L.w2.p, static_cast<uint64_t>(nslots) * c->d, c->ff, 256);
  L.tmB1h = make_kmajor_map(L.w13.p, static_cast<uint64_t>(nslots) * 2 * c->ff, c->d, 128);
  L.tmB2h = make_kmajor_map(L.w2.p, static_cast<uint64_t>(nslots) * c->d, c->ff, 128);
  L.expert_loaded.assign(c->E, 0);
}

// Enqueue one forward.  Three planning paths:
//   local : G == 1 — the device builds the dispatch plan from its own
//           histogram (plan_local_kernel);
//   ahead : peer-memory exchange (G > 1, bf16) with the placement decided
//           before the layer (FIXED, or PREDICTED planned d layers ahead) —
//           the device builds the exchange plan from the gathered histograms
//           (plan_exchange_kernel);
//   host  : otherwise (NCCL chunk lists, MOE_PLAN_SYNC or a bootstrap layer
//           at G > 1) — one host round trip: counts down, plan up.
// local / ahead never wait for the host: the MoEless planner bookkeeping
// (scale/place on the actual loads for SYNC, registry, predictor accuracy,
// planning layer l + d) runs when the next call flushes it, as soon as this
// forward's histogram is in mapped host memory.  Those two paths are also
// capturable as one CUDA graph (capturing = true: external event nodes, no
// per-call timing events).
template <class Mark>
void enqueue_forward(moe_ctx* c, Layer& L, int layer, const uint16_t* x, int T, uint16_t* y, int plan_mode,
                     long iteration, cudaStream_t s, bool with_pred, int stride, cudaEvent_t x_consumed, bool ahead,
                     bool capturing, Mark&& mark) {
  const unsigned rec = capturing ? cudaEventRecordExternal : cudaEventRecordDefault;
  const bool deferred = c->G == 1 || ahead;
  // single GPU, bf16, 1-SM K4: GEMM1 gathers its A rows from x (TMA gather4)
  // and the dispatch kernel only ranks — no permuted copy of the tokens
  const bool gather = c->gather && c->G == 1 && !c->fp32 && (c->gemm_variant == 0 || c->gemm_variant == 1) && T > 0;
  // single GPU, bf16, 1-SM K4: the combine runs inside GEMM2's epilogue
  const bool fused = c->fuse_combine && c->G == 1 && !c->fp32 && (c->gemm_variant == 0 || c->gemm_variant == 1);
  if (gather && (c->tmX_ptr != x || c->tmX_T != T)) {
    c->tmX = make_kmajor_map(x, T, c->d, 1);
    c->tmX_ptr = x;
    c->tmX_T = T;
  }
  mark(0);
  stage_gate(c, L, x, T, s, with_pred ? c->counts.p + c->E : nullptr);
  if (c->G > 1 && c->p2p) {
    // every rank reads every histogram from its owner's slab
    CU_CHECK(launch_p2p_counts(c->peers, c->G, c->rank, stride, c->epoch_dev.p, c->p2p_timeout_ns, c->p2p_err,
                               c->counts_all.p, s));
    if (c->placed && !c->peers_ready) {
      // every rank has entered its first forward, so every home expert is
      // loaded: weight copies from peers may start from here on
      CU_CHECK(cudaEventRecord(c->ev_peers_ready, s));
      CU_CHECK(cudaStreamWaitEvent(c->wstream, c->ev_peers_ready, 0));
      c->peers_ready = true;
      for (size_t l = 0; l < c->layers.size(); ++l) issue_weight_copies(c, static_cast<int>(l));
    }
    CU_CHECK(launch_small_copy(c->h_counts, c->counts_all.p, pad16(sizeof(int32_t) * c->G * stride), s));
  } else if (c->G > 1) {
    require(c->desc.exchange_mode == MOE_EXCHANGE_NCCL, "staged API required for external exchange");
    g_nccl.check(g_nccl.AllGather(c->counts.p, c->counts_all.p, stride, ncclInt32, c->comm, s), "ncclAllGather");
    CU_CHECK(launch_small_copy(c->h_counts, c->counts_all.p, pad16(sizeof(int32_t) * c->G * stride), s));
  } else {
    CU_CHECK(launch_small_copy(c->h_counts, c->counts.p, pad16(sizeof(int32_t) * stride), s));
  }
  if (deferred) {
    CU_CHECK(cudaEventRecordWithFlags(c->ev_counts, s, rec));
    mark(1);
    if (c->G == 1)
      CU_CHECK(launch_plan_local(c->counts.p, c->E, c->dplan.p, s));
    else
      CU_CHECK(launch_plan_exchange(c->counts_all.p, stride, c->G, c->rank, L.ptab.p, c->dplan.p, s));
    mark(2);
    stage_dispatch(c, x, T, s, /*upload_plan=*/false, gather, fused);
  } else {
    mark(1);
    CU_CHECK(cudaStreamSynchronize(s));  // the host plans on the real histogram
    check_p2p(c);
    stage_plan(c, layer, plan_mode, iteration, c->h_counts, stride);
    mark(2);
    stage_dispatch(c, x, T, s);  // uploads the plan; P2P rows land in their owners' buffers
  }
  // x is not read after dispatch (after GEMM1 when GEMM1 gathers from it)
  if (x_consumed && !gather) CU_CHECK(cudaEventRecordWithFlags(x_consumed, s, rec));
  mark(3);
  stage_exchange(c, true, s);
  mark(4);
  // rows only sizes the fp32 SwiGLU pass (bf16 GEMMs read the device plan)
  const int64_t rows = c->G == 1 ? static_cast<int64_t>(T) * c->k : (ahead ? c->rows_cap : c->plan.rows_local);
  const int gslot = static_cast<int>(c->gemm_seq % moe_ctx::kGemmRing);
  if (c->placed && L.wready_valid) CU_CHECK(cudaStreamWaitEvent(s, L.ev_wready, 0));  // cold replicas copied in
  if (!capturing) CU_CHECK(cudaEventRecord(c->gemm_ev[gslot][0], s));
  launch_ffn_gemm(c, layer, 0, s, rows, gather);
  // (with PDL, an event between the GEMMs would serialise them: GEMM1+GEMM2 is
  // then timed as one interval, reported as GEMM1 with GEMM2 = 0)
  if (!capturing && !c->use_pdl) CU_CHECK(cudaEventRecord(c->gemm_ev[gslot][1], s));
  mark(5);
  launch_ffn_gemm(c, layer, 1, s, rows, false, fused ? y : nullptr);
  // (after GEMM2, not between the GEMMs: an event there would serialise the PDL pair)
  if (x_consumed && gather) CU_CHECK(cudaEventRecordWithFlags(x_consumed, s, rec));
  if (c->placed) {  // the layer's slots may be overwritten once these GEMMs are done
    CU_CHECK(cudaEventRecord(L.ev_used, s));
    L.used_recorded = true;
  }
  if (!capturing) {
    CU_CHECK(cudaEventRecord(c->gemm_ev[gslot][2], s));
    c->gemm_rows[gslot] = ahead ? -1 : rows;  // "ahead": filled in when the plan is flushed
    ++c->gemm_seq;
  }
  mark(6);
  stage_exchange(c, false, s);
  mark(7);
  if (!fused) stage_combine(c, y, T, s);
  mark(8);
  if (deferred && !capturing) c->pending = PendingPlan{true, layer, plan_mode, iteration, stride, ahead ? gslot : -1};
}

void forward_device(moe_ctx* c, int layer, const uint16_t* x, int T, uint16_t* y, int plan_mode, long iteration,
                    moe_layer_stats* st, cudaStream_t s, cudaEvent_t x_consumed = nullptr) {
  Layer& L = layer_at(c, layer);
  CU_CHECK(cudaSetDevice(c->desc.device));  // callers may drive ranks from several host threads
  require(T >= 0 && T <= c->Tmax, "token count exceeds max_tokens");
  c->cur_T = T;
  require(plan_mode == MOE_PLAN_FIXED || plan_mode == MOE_PLAN_SYNC || plan_mode == MOE_PLAN_PREDICTED,
          "unknown plan mode");
  for (int e = 0; e < c->E; ++e)
    if (!L.w13.p || !L.expert_loaded[e]) throw std::invalid_argument("expert weights not loaded for layer");
  if (c->p2p) {
    require(c->p2p_ready, "moe_p2p_import must be called before a peer-memory forward");
    check_p2p(c);
  }
  EventSet& ev = c->events;
  const bool timed = st != nullptr;
  flush_pending_plan(c);  // the previous call's deferred planner work
  // the fused predictor (K2) runs when the layer has predictor weights: its
  // histograms follow the gate's in the same counts buffer
  const bool with_pred = c->n_pred > 0 && L.has_pred_weights;
  const int stride = with_pred ? c->count_stride : c->E;
  const bool ahead = c->G > 1 && c->p2p && !c->fp32 &&
                     (plan_mode == MOE_PLAN_FIXED || (plan_mode == MOE_PLAN_PREDICTED && L.plan_for == iteration));
  if (ahead) ensure_placement(c, layer);
  if (c->use_graphs && !timed && (c->G == 1 || ahead) && !c->placed) {
    // Replay the layer's whole device sequence (8-14 kernels) as one CUDA
    // graph: captured once per (layer, tokens, buffers), then launched with a
    // single call — the launch-bound decode regime pays one launch, not ten.
    const GraphKey key{layer, T, x, y, x_consumed, with_pred};
    auto it = c->graphs.find(key);
    if (it == c->graphs.end()) {
      CU_CHECK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
      enqueue_forward(c, L, layer, x, T, y, plan_mode, iteration, s, with_pred, stride, x_consumed, ahead, true,
                      [](int) {});
      cudaGraph_t g = nullptr;
      CU_CHECK(cudaStreamEndCapture(s, &g));
      cudaGraphExec_t ex = nullptr;
      const cudaError_t e = cudaGraphInstantiate(&ex, g, 0);
      cudaGraphDestroy(g);
      CU_CHECK(e);
      it = c->graphs.emplace(key, ex).first;
    }
    CU_CHECK(cudaGraphLaunch(it->second, s));
    c->pending = PendingPlan{true, layer, plan_mode, iteration, stride, -1};
    return;
  }
  enqueue_forward(c, L, layer, x, T, y, plan_mode, iteration, s, with_pred, stride, x_consumed, ahead, false,
                  [&](int i) {
                    if (timed) CU_CHECK(cudaEventRecord(ev.ev[i], s));
                  });
  if (timed) {
    CU_CHECK(cudaEventSynchronize(ev.ev[8]));
    flush_pending_plan(c);
    st->gate_ms = ev.ms(0, 1);
    st->plan_ms = ev.ms(1, 2);
    st->dispatch_ms = ev.ms(2, 3);
    st->a2a_dispatch_ms = ev.ms(3, 4);
    st->gemm1_ms = ev.ms(4, 5);
    st->gemm2_ms = ev.ms(5, 6);
    st->a2a_combine_ms = ev.ms(6, 7);
    st->combine_ms = ev.ms(7, 8);
    st->forward_ms = ev.ms(0, 8);
    st->compute_ms = st->gemm1_ms + st->gemm2_ms;
    st->comm_ms = 0.5 * (st->a2a_dispatch_ms + st->a2a_combine_ms);
    st->replica_count = static_cast<int>(L.rep_gpu.size());
    st->mem_mb = st->replica_count * (3.0 * c->d * c->ff * 2 / 1e6);
    st->rows_local = c->plan.rows_local;
    st->rows_sent = c->plan.rows_send;
    st->warm_count = L.warm;
    st->cold_count = L.cold;
    st->predictor_accuracy = L.last_accuracy;
    st->plan_source = L.plan_source;
    st->weight_copies = L.copies_last;
    st->weight_hits = L.hits_last;
    st->weight_copy_mb = L.copies_last * static_cast<double>(c->w13_slot_bytes + c->w2_slot_bytes) / 1e6;
    st->weight_copy_ms = 0.0;
    if (L.wready_timed && L.wready_valid) {
      float ms = 0.0f;
      CU_CHECK(cudaEventSynchronize(L.ev_wready));
      CU_CHECK(cudaEventElapsedTime(&ms, L.ev_wstart, L.ev_wready));
      st->weight_copy_ms = ms;
    }
    for (int e = 0; e < c->E && e < 256; ++e) st->counts[e] = c->h_counts[static_cast<size_t>(c->rank) * c->E + e];
  }
}

}  // namespace

// ==================================================================== C ABI
extern "C" {

const char* moe_last_error(void) { return g_last_error.c_str(); }
const char* moe_version(void) { return "moe_b200 0.1.0 (sm_100a)"; }

int moe_nccl_unique_id(void* out128) {
  return guarded([&] {
    require(out128 != nullptr, "null argument");
    g_nccl.load();
    ncclUniqueId id;
    g_nccl.check(g_nccl.GetUniqueId(&id), "ncclGetUniqueId");
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(out128, &id, sizeof(id));
  });
}

int moe_ctx_create(const moe_ctx_desc* desc, moe_ctx** out) {
  return guarded([&] {
    require(desc && out, "null argument");
    const moe_ctx_desc& D = *desc;
    require(D.num_layers >= 1, "num_layers must be >= 1");
    require(D.num_experts >= 1 && D.num_experts <= kMaxExperts, "num_experts out of range");
    require(D.top_k >= 1 && D.top_k <= D.num_experts && D.top_k <= 8 && (D.top_k <= 2 || D.top_k % 2 == 0),
            "top_k must be in {1,2,4,6,8} and <= num_experts");
    require(D.d_model % 256 == 0 && D.d_model > 0, "d_model must be a positive multiple of 256");
    require(D.d_ff % 128 == 0 && D.d_ff > 0, "d_ff must be a positive multiple of 128");
    require(D.max_tokens >= 1, "max_tokens must be >= 1");
    require(D.world_size >= 1 && D.rank >= 0 && D.rank < D.world_size, "bad world_size / rank");
    require(D.num_experts * (1 + std::max(0, D.num_predictor_targets)) <= 256, "too many predictor targets");
    int ndev = 0;
    CU_CHECK(cudaGetDeviceCount(&ndev));
    require(D.device >= 0 && D.device < ndev, "device ordinal out of range");
    CU_CHECK(cudaSetDevice(D.device));
    cudaDeviceProp prop;
    CU_CHECK(cudaGetDeviceProperties(&prop, D.device));
    if (prop.major != 10) throw Status(MOE_ECUDA, "moe_b200 requires an sm_100 (Blackwell) device");
    auto c = std::make_unique<moe_ctx>();
    c->desc = D;
    c->E = D.num_experts;
    c->k = D.top_k;
    c->d = D.d_model;
    c->ff = D.d_ff;
    c->G = D.world_size;
    c->rank = D.rank;
    c->Tmax = D.max_tokens;
    c->n_pred = std::max(0, D.num_predictor_targets);
    c->pred_distance = D.predictor_distance > 0 ? D.predictor_distance : 1;
    c->use_graphs = D.use_cuda_graphs != 0;
    if (const char* v = std::getenv("MOE_CUDA_GRAPHS")) c->use_graphs = std::string(v) == "1";
    c->num_sms = prop.multiProcessorCount;
    if (const char* v = std::getenv("MOE_GEMM_SCHED")) c->dyn_sched = std::string(v) == "dynamic";
    if (const char* v = std::getenv("MOE_PDL")) c->use_pdl = std::string(v) != "0";
    if (const char* v = std::getenv("MOE_GATHER")) c->gather = std::string(v) == "1";
    if (const char* v = std::getenv("MOE_FUSED_COMBINE")) c->fuse_combine = std::string(v) == "1";
    if (const char* v = std::getenv("MOE_GEMM_GROUP_M")) std::sscanf(v, "%d,%d", &c->group_m[0], &c->group_m[1]);
    if (const char* v = std::getenv("MOE_GEMM_VARIANT")) {
      const std::string s(v);
      c->gemm_variant = s == "1sm" ? 1 : (s == "2sm" ? 2 : (s == "m256" ? 3 : 0));
    }
    c->registry = moeless::ReplicaRegistry(std::max(0, D.keep_alive_iters));
    c->layers.resize(D.num_layers);
    require(D.precision == MOE_PRECISION_BF16 || D.precision == MOE_PRECISION_FP32, "unknown precision");
    c->fp32 = D.precision == MOE_PRECISION_FP32;
    c->elem = c->fp32 ? 2 : 1;
    require(!c->fp32 || c->n_pred == 0, "the fp32 mode has no fused predictor");
    require(D.residency == MOE_RESIDENCY_ALL || D.residency == MOE_RESIDENCY_PLACED, "unknown residency");
    c->placed = D.residency == MOE_RESIDENCY_PLACED && c->G > 1;  // G == 1: every expert is home
    if (c->placed) {
      require(D.exchange_mode == MOE_EXCHANGE_P2P,
              "MOE_RESIDENCY_PLACED needs the peer-memory exchange (MOE_EXCHANGE_P2P): replicas are copied "
              "from their home rank over NVLink");
      require(!c->fp32, "MOE_RESIDENCY_PLACED supports the bf16 path only");
      c->home_slots = (c->E + c->G - 1) / c->G;
      // the same layout on every rank (peers address each other's slots)
      const int max_cache = c->E - c->E / c->G;
      const double mem = D.expert_mem_mb > 0 ? D.expert_mem_mb : 3.0 * c->d * c->ff * 2 / 1e6;
      int cache = D.replica_slots > 0 ? D.replica_slots
                                      : static_cast<int>(std::min<double>(max_cache, std::floor(
                                            (D.gpu_mem_capacity_mb > 0 ? D.gpu_mem_capacity_mb : 180000.0) / mem)));
      c->cache_slots = std::max(1, std::min(cache, max_cache));
      c->slots = c->home_slots + c->cache_slots;
      c->w13_slot_bytes = static_cast<size_t>(2) * c->ff * c->d * 2;
      c->w2_slot_bytes = static_cast<size_t>(c->d) * c->ff * 2;
      c->layer_wbytes = static_cast<size_t>(c->slots) * (c->w13_slot_bytes + c->w2_slot_bytes);
    }
    CU_CHECK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    // load every kernel now, not lazily at first launch (see preload_*)
    CU_CHECK(preload_gate_kernels());
    CU_CHECK(preload_dispatch_kernels());
    CU_CHECK(preload_gemm_kernels());
    CU_CHECK(preload_fp32_kernels());
    CU_CHECK(preload_p2p_kernels());
    const int64_t assign = static_cast<int64_t>(c->Tmax) * c->k;
    c->rows_cap = assign * c->G;  // worst case: every rank routes everything here
    c->send_cap = c->G > 1 ? assign : 1;
    const int nblk = gate_num_blocks(c->Tmax);
    c->ids.alloc(assign);
    c->wts.alloc(assign);
    c->row_code.alloc(assign);
    c->count_stride = c->E * (1 + c->n_pred);  // [gate E | predictor n_pred x E]
    c->counts.alloc(pad16(sizeof(int32_t) * c->count_stride) / 4);
    c->counts_all.alloc(pad16(sizeof(int32_t) * c->count_stride * c->G) / 4);
    c->pred_counts.alloc(static_cast<size_t>(c->E) * std::max(1, c->n_pred));
    c->block_counts.alloc(static_cast<size_t>(nblk) * c->E);
    c->block_pre.alloc(static_cast<size_t>(nblk) * c->E);
    // row buffers in 16-bit units: one row = d_model * elem units (elem 2 for fp32)
    c->xw = c->d * c->elem;
    c->xp.alloc(static_cast<size_t>(c->rows_cap) * c->xw);
    c->perm_src.alloc(static_cast<size_t>(c->rows_cap));
    c->row_owner.alloc(static_cast<size_t>(c->rows_cap));
    c->comb_cnt.alloc(static_cast<size_t>(c->Tmax) * std::max(1, c->d / 256));
    CU_CHECK(cudaMemset(c->comb_cnt.p, 0, c->comb_cnt.n * sizeof(int32_t)));
    c->h.alloc(static_cast<size_t>(c->rows_cap) * c->ff * c->elem);
    c->yp.alloc(static_cast<size_t>(c->rows_cap) * c->xw);
    c->send.alloc(static_cast<size_t>(c->send_cap) * c->xw);
    c->ret.alloc(static_cast<size_t>(c->send_cap) * c->xw);
    if (c->G > 1 && D.exchange_mode == MOE_EXCHANGE_P2P) {
      // one exported slab: flags | counts | received rows (xp) | expert outputs (yp)
      require(c->G <= kMaxRanks, "the peer-memory exchange supports up to 8 ranks");
      c->p2p = true;
      auto up = [](size_t b) { return (b + 4095) & ~size_t(4095); };
      const size_t rows_bytes = static_cast<size_t>(c->rows_cap) * c->xw * 2;
      c->off_flags = 0;
      c->off_counts = up(sizeof(uint32_t) * kFlagKinds * kMaxRanks);
      c->off_xp = c->off_counts + up(sizeof(int32_t) * c->count_stride);
      c->off_yp = c->off_xp + up(rows_bytes);
      c->off_weights = c->off_yp + up(rows_bytes);
      // MOE_RESIDENCY_PLACED: every layer's weight slots live in the slab too
      c->slab.alloc(c->off_weights + (c->placed ? c->layer_wbytes * c->layers.size() : 0));
      CU_CHECK(cudaMemset(c->slab.p, 0, c->off_xp));  // flags start at epoch 0
      c->counts.view(c->slab.p + c->off_counts, pad16(sizeof(int32_t) * c->count_stride) / 4);
      c->xp.view(c->slab.p + c->off_xp, static_cast<size_t>(c->rows_cap) * c->xw);
      c->yp.view(c->slab.p + c->off_yp, static_cast<size_t>(c->rows_cap) * c->xw);
      CU_CHECK(cudaHostAlloc(&c->p2p_err, sizeof(int) * 4, cudaHostAllocMapped));
      c->dispatch_counter.alloc(4);
      CU_CHECK(cudaMemset(c->dispatch_counter.p, 0, 16));
      c->epoch_dev.alloc(4);
      CU_CHECK(cudaMemset(c->epoch_dev.p, 0, 16));
      *c->p2p_err = 0;
      if (c->placed) {
        CU_CHECK(cudaStreamCreateWithFlags(&c->wstream, cudaStreamNonBlocking));
        CU_CHECK(cudaEventCreateWithFlags(&c->ev_peers_ready, cudaEventDisableTiming));
      }
      if (const char* v = std::getenv("MOE_P2P_TIMEOUT_MS")) c->p2p_timeout_ns = std::strtoull(v, nullptr, 10) * 1000000ull;
    }
    c->dplan.alloc(1);
    c->gemm_sched.alloc(4);
    CU_CHECK(cudaMemset(c->gemm_sched.p, 0, 4 * sizeof(int)));
    {  // split-K gate scratch: <= 296 (block, split) CTAs x 32 tokens x padded logits
      int nt = 1;
      while (8 * nt < c->count_stride) nt *= 2;
      c->gate_partial.alloc(static_cast<size_t>(296) * 32 * 8 * nt);
    }
    if (c->fp32) {
      c->gu_f32.alloc(static_cast<size_t>(c->rows_cap) * 2 * c->ff);  // GEMM1 output before SwiGLU
    } else {
      c->tmA1 = make_kmajor_map(c->xp.p, c->rows_cap, c->d, 128);
      c->tmA2 = make_kmajor_map(c->h.p, c->rows_cap, c->ff, 128);
      c->tmA1w = make_kmajor_map(c->xp.p, c->rows_cap, c->d, 256);
      c->tmA2w = make_kmajor_map(c->h.p, c->rows_cap, c->ff, 256);
    }
    // mapped pinned control buffers, read/written by small SM copies (UVA pointers)
    CU_CHECK(cudaHostAlloc(&c->hplan, sizeof(DevPlan), cudaHostAllocMapped));
    CU_CHECK(cudaHostAlloc(&c->h_counts, pad16(sizeof(int32_t) * c->count_stride * c->G), cudaHostAllocMapped));
    c->events.create();
    CU_CHECK(cudaEventCreateWithFlags(&c->ev_counts, cudaEventDisableTiming));
    for (auto& tri : c->gemm_ev)
      for (cudaEvent_t& e : tri) CU_CHECK(cudaEventCreate(&e));
    if (c->G > 1 && D.exchange_mode == MOE_EXCHANGE_NCCL) {
      require(D.nccl_unique_id != nullptr, "nccl_unique_id required for world_size > 1");
      g_nccl.load();
      ncclUniqueId id;
      std::memcpy(&id, D.nccl_unique_id, sizeof(id));
      g_nccl.check(g_nccl.CommInitRank(&c->comm, c->G, id, c->rank), "ncclCommInitRank");
    }
    *out = c.release();
  });
}

int moe_ctx_destroy(moe_ctx* c) {
  return guarded([&] {
    if (!c) return;
    cudaSetDevice(c->desc.device);
    cudaStreamSynchronize(c->stream);
    if (c->comm) g_nccl.CommDestroy(c->comm);
    for (void* q : c->ipc_opened) cudaIpcCloseMemHandle(q);
    if (c->wstream) cudaStreamSynchronize(c->wstream);
    for (Layer& L : c->layers) {
      if (L.h_ptab) cudaFreeHost(L.h_ptab);
      for (cudaEvent_t e : {L.ev_ptab, L.ev_used, L.ev_wstart, L.ev_wready})
        if (e) cudaEventDestroy(e);
    }
    if (c->ev_peers_ready) cudaEventDestroy(c->ev_peers_ready);
    if (c->wstream) cudaStreamDestroy(c->wstream);
    if (c->p2p_err) cudaFreeHost(c->p2p_err);
    c->events.destroy();
    if (c->hplan) cudaFreeHost(c->hplan);
    if (c->h_counts) cudaFreeHost(c->h_counts);
    if (c->wg_stage) cudaFreeHost(c->wg_stage);
    if (c->ev_wg_staged) cudaEventDestroy(c->ev_wg_staged);
    if (c->ev_counts) cudaEventDestroy(c->ev_counts);
    for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second);
    for (auto& tri : c->gemm_ev)
      for (cudaEvent_t e : tri)
        if (e) cudaEventDestroy(e);
    if (c->h2d) {
      cudaStreamSynchronize(c->h2d);
      cudaStreamSynchronize(c->d2h);
      for (int i = 0; i < 2; ++i)
        for (cudaEvent_t e : {c->ev_x_ready[i], c->ev_x_free[i], c->ev_y_ready[i], c->ev_done[i]})
          if (e) cudaEventDestroy(e);
      for (cudaEvent_t e : c->ev_ticket)
        if (e) cudaEventDestroy(e);
      cudaStreamDestroy(c->h2d);
      cudaStreamDestroy(c->d2h);
    }
    cudaStreamDestroy(c->stream);
    delete c;
  });
}

int moe_ctx_stream(moe_ctx* c, void** s) {
  return guarded([&] {
    require(c && s, "null argument");
    *s = c->stream;
  });
}

int moe_ctx_sync(moe_ctx* c) {
  return guarded([&] {
    require(c, "null context");
    CU_CHECK(cudaStreamSynchronize(c->stream));
    flush_pending_plan(c);
  });
}

int moe_p2p_export(moe_ctx* c, moe_p2p_handle* out) {
  return guarded([&] {
    require(c && out, "null argument");
    require(c->p2p, "context was not created with MOE_EXCHANGE_P2P and world_size > 1");
    static_assert(sizeof(moe_p2p_handle) == 192, "moe_p2p_handle layout");
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "cudaIpcMemHandle_t is 64 bytes");
    moe_p2p_handle h{};
    cudaIpcMemHandle_t ipc;
    CU_CHECK(cudaIpcGetMemHandle(&ipc, c->slab.p));
    std::memcpy(h.ipc, &ipc, sizeof(ipc));
    h.pid = static_cast<uint64_t>(getpid());
    h.base = reinterpret_cast<uint64_t>(c->slab.p);
    h.bytes = c->slab.n;
    h.off_flags = c->off_flags;
    h.off_counts = c->off_counts;
    h.off_xp = c->off_xp;
    h.off_yp = c->off_yp;
    h.device = c->desc.device;
    h.rank = c->rank;
    h.world_size = c->G;
    h.version = 1;
    h.off_weights = c->off_weights;
    h.weight_bytes = c->placed ? c->layer_wbytes * c->layers.size() : 0;
    *out = h;
  });
}

int moe_p2p_import(moe_ctx* c, const moe_p2p_handle* hs, int n) {
  return guarded([&] {
    require(c && hs, "null argument");
    require(c->p2p, "context was not created with MOE_EXCHANGE_P2P and world_size > 1");
    require(!c->p2p_ready, "peer slabs already imported");
    require(n == c->G, "need one handle per rank");
    CU_CHECK(cudaSetDevice(c->desc.device));
    for (int g = 0; g < n; ++g) {
      const moe_p2p_handle& h = hs[g];
      require(h.version == 1 && h.rank == g && h.world_size == c->G, "handle " + std::to_string(g) +
                                                                          " is not rank " + std::to_string(g) +
                                                                          " of this world");
      require(h.bytes == c->slab.n && h.off_xp == c->off_xp && h.off_yp == c->off_yp &&
                  h.off_counts == c->off_counts && h.off_weights == c->off_weights &&
                  h.weight_bytes == (c->placed ? c->layer_wbytes * c->layers.size() : 0),
              "rank " + std::to_string(g) + " was created with a different shape");
      uint8_t* base = nullptr;
      if (g == c->rank) {
        base = c->slab.p;
      } else if (h.pid == static_cast<uint64_t>(getpid())) {
        // same process (ranks driven by threads): the pointer is valid here; a
        // different device needs peer access
        if (h.device != c->desc.device) {
          int ok = 0;
          CU_CHECK(cudaDeviceCanAccessPeer(&ok, c->desc.device, h.device));
          require(ok != 0, "device " + std::to_string(c->desc.device) + " cannot access device " +
                               std::to_string(h.device));
          const cudaError_t e = cudaDeviceEnablePeerAccess(h.device, 0);
          if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
          else CU_CHECK(e);
        }
        base = reinterpret_cast<uint8_t*>(h.base);
      } else {
        cudaIpcMemHandle_t ipc;
        std::memcpy(&ipc, h.ipc, sizeof(ipc));
        void* q = nullptr;
        CU_CHECK(cudaIpcOpenMemHandle(&q, ipc, cudaIpcMemLazyEnablePeerAccess));
        c->ipc_opened.push_back(q);
        base = static_cast<uint8_t*>(q);
      }
      c->peers.flags[g] = reinterpret_cast<uint32_t*>(base + h.off_flags);
      c->peers.counts[g] = reinterpret_cast<const int32_t*>(base + h.off_counts);
      c->xp_targets.base[g] = base + h.off_xp;
      c->peer_base[g] = base;
      c->yp_targets.base[g] = base + h.off_yp;
    }
    c->p2p_ready = true;
  });
}

namespace {
// elem: 16-bit units per element of the caller's arrays (1 bf16, 2 fp32)
void load_expert_impl(moe_ctx* c, int layer, int expert, const void* w1v, const void* w3v, const void* w2v,
                      int elem) {
  Layer& L = layer_at(c, layer);
  require(elem == c->elem, elem == 2 ? "fp32 weights need a MOE_PRECISION_FP32 context"
                                     : "bf16 weights need a MOE_PRECISION_BF16 context");
  require(expert >= 0 && expert < c->E, "expert out of range");
  require(w1v && w3v && w2v, "null weight pointer");
  ensure_pools(c, L);
  int slot = expert;
  if (c->placed) {
    if (expert % c->G != c->rank) {  // not home here: replicas are copied from the home rank
      L.expert_loaded[expert] = 1;
      return;
    }
    slot = expert / c->G;
  }
  const uint16_t* w1 = static_cast<const uint16_t*>(w1v);
  const uint16_t* w3 = static_cast<const uint16_t*>(w3v);
  const uint16_t* w2 = static_cast<const uint16_t*>(w2v);
  // W13 pool: per 128-row block b of the expert, rows [W1[b*128..], W3[b*128..]]
  const size_t row = static_cast<size_t>(c->d) * elem;  // one weight row in 16-bit units
  uint16_t* base = L.w13.p + static_cast<size_t>(slot) * 2 * c->ff * row;
  for (int b = 0; b < c->ff / 128; ++b) {
    CU_CHECK(cudaMemcpyAsync(base + static_cast<size_t>(b) * 256 * row, w1 + static_cast<size_t>(b) * 128 * row,
                             128 * row * 2, cudaMemcpyHostToDevice, c->stream));
    CU_CHECK(cudaMemcpyAsync(base + (static_cast<size_t>(b) * 256 + 128) * row, w3 + static_cast<size_t>(b) * 128 * row,
                             128 * row * 2, cudaMemcpyHostToDevice, c->stream));
  }
  CU_CHECK(cudaMemcpyAsync(L.w2.p + static_cast<size_t>(slot) * c->d * c->ff * elem, w2,
                           static_cast<size_t>(c->d) * c->ff * 2 * elem, cudaMemcpyHostToDevice, c->stream));
  CU_CHECK(cudaStreamSynchronize(c->stream));
  L.expert_loaded[expert] = 1;
}
}  // namespace

int moe_load_expert_weights(moe_ctx* c, int layer, int expert, const uint16_t* w1, const uint16_t* w3,
                            const uint16_t* w2) {
  return guarded([&] { load_expert_impl(c, layer, expert, w1, w3, w2, 1); });
}

int moe_load_expert_weights_f32(moe_ctx* c, int layer, int expert, const float* w1, const float* w3,
                                const float* w2) {
  return guarded([&] { load_expert_impl(c, layer, expert, w1, w3, w2, 2); });
}

namespace {
void set_gate_impl(moe_ctx* c, int layer, const void* wg, int elem) {
  Layer& L = layer_at(c, layer);
  require(wg != nullptr, "null gate weights");
  require(elem == c->elem, "gate weight precision does not match the context");
  if (!L.wg.p) {
    L.wg.alloc(static_cast<size_t>(c->E) * c->d * (1 + c->n_pred) * elem);
    CU_CHECK(cudaMemsetAsync(L.wg.p, 0, L.wg.n * 2, c->stream));
  }
  // Stream-ordered update through a pinned staging buffer: forwards already
  // enqueued keep the old weights, later ones see the new — no device sync.
  const size_t bytes = static_cast<size_t>(c->E) * c->d * 2 * elem;
  if (c->wg_stage && c->wg_stage_bytes < bytes) {
    CU_CHECK(cudaEventSynchronize(c->ev_wg_staged));
    CU_CHECK(cudaFreeHost(c->wg_stage));
    c->wg_stage = nullptr;
  }
  if (!c->wg_stage) {
    CU_CHECK(cudaHostAlloc(&c->wg_stage, bytes, cudaHostAllocMapped));
    c->wg_stage_bytes = bytes;
    if (!c->ev_wg_staged) CU_CHECK(cudaEventCreateWithFlags(&c->ev_wg_staged, cudaEventDisableTiming));
  } else {
    CU_CHECK(cudaEventSynchronize(c->ev_wg_staged));  // previous upload has left the staging buffer
  }
  std::memcpy(c->wg_stage, wg, bytes);
  CU_CHECK(launch_small_copy(L.wg.p, c->wg_stage, bytes, c->stream));
  CU_CHECK(cudaEventRecord(c->ev_wg_staged, c->stream));
  L.has_gate = true;
}
}  // namespace

int moe_set_gate_weights_f32(moe_ctx* c, int layer, const float* wg) {
  return guarded([&] { set_gate_impl(c, layer, wg, 2); });
}

int moe_set_gate_weights(moe_ctx* c, int layer, const uint16_t* wg) {
  return guarded([&] { set_gate_impl(c, layer, wg, 1); });
}

int moe_set_predictor_weights(moe_ctx* c, int layer, int slot, const uint16_t* wp) {
  return guarded([&] {
    Layer& L = layer_at(c, layer);
    require(slot >= 0 && slot < c->n_pred, "predictor slot out of range");
    require(wp != nullptr, "null predictor weights");
    if (!L.wg.p) {
      L.wg.alloc(static_cast<size_t>(c->E) * c->d * (1 + c->n_pred));
      CU_CHECK(cudaMemsetAsync(L.wg.p, 0, L.wg.n * 2, c->stream));
    }
    CU_CHECK(cudaStreamSynchronize(c->stream));  // no enqueued forward may see a half-written gate
    CU_CHECK(cudaMemcpy(L.wg.p + static_cast<size_t>(1 + slot) * c->E * c->d, wp, static_cast<size_t>(c->E) * c->d * 2,
                        cudaMemcpyHostToDevice));
    L.has_pred_weights = true;
  });
}

int moe_set_placement(moe_ctx* c, int layer, const int32_t* rc, const int32_t* rg) {
  return guarded([&] {
    Layer& L = layer_at(c, layer);
    require(rc && rg, "null placement");
    int total = 0;
    for (int e = 0; e < c->E; ++e) {
      require(rc[e] >= 1, "expert " + std::to_string(e) + " has no replica");
      total += rc[e];
    }
    require(total <= kMaxReplicas, "too many replicas in one layer");
    for (int i = 0; i < total; ++i)
      require(rg[i] >= 0 && rg[i] < c->G,
              "replica placed on invalid GPU " + std::to_string(rg[i]));
    std::vector<int32_t> old_counts = L.rep_counts, old_gpu = L.rep_gpu;
    const bool had = L.has_placement;
    L.rep_counts.assign(rc, rc + c->E);
    L.rep_gpu.assign(rg, rg + total);
    try {
      placement_changed(c, layer);
    } catch (...) {  // an infeasible placement leaves the previous one in force
      L.rep_counts.swap(old_counts);
      L.rep_gpu.swap(old_gpu);
      L.has_placement = had;
      throw;
    }
  });
}

int moe_gate_topk(moe_ctx* c, int layer, const uint16_t* x, int T, int32_t* ids, float* w, int32_t* counts,
                  int32_t* pred_counts, void* stream) {
  return guarded([&] {
    Layer& L = layer_at(c, layer);
    require(T >= 0 && T <= c->Tmax, "token count exceeds max_tokens");
    require(x && ids && w && counts, "null buffer");
    cudaStream_t s = pick(c, stream);
    require(L.has_gate, "gate weights not set for layer");
    CU_CHECK(cudaMemsetAsync(counts, 0, sizeof(int32_t) * c->E, s));
    if (pred_counts && c->n_pred) CU_CHECK(cudaMemsetAsync(pred_counts, 0, sizeof(int32_t) * c->E * c->n_pred, s));
    CU_CHECK(launch_gate_topk(reinterpret_cast<const __nv_bfloat16*>(x), T, c->d,
                              reinterpret_cast<const __nv_bfloat16*>(L.wg.p), c->E, pred_counts ? c->n_pred : 0, c->k,
                              ids, w, counts, c->block_counts.p, pred_counts ? pred_counts : c->pred_counts.p,
                              c->gate_partial.p, s));
  });
}

int moe_predict_loads(moe_ctx* c, int layer, const uint16_t* x, int T, int32_t* pred_counts, void* stream) {
  return guarded([&] {
    Layer& L = layer_at(c, layer);
    require(c->n_pred > 0, "context has no predictor targets");
    require(T >= 0 && T <= c->Tmax, "token count exceeds max_tokens");
    require(x && pred_counts, "null buffer");
    cudaStream_t s = pick(c, stream);
    require(L.has_gate, "gate weights not set for layer");
    // the gate rows ride along (they are in the same stacked matrix); their
    // outputs go to the ctx scratch so the caller's ids are untouched
    CU_CHECK(cudaMemsetAsync(pred_counts, 0, sizeof(int32_t) * c->E * c->n_pred, s));
    CU_CHECK(cudaMemsetAsync(c->counts.p, 0, sizeof(int32_t) * c->E, s));
    CU_CHECK(launch_gate_topk(reinterpret_cast<const __nv_bfloat16*>(x), T, c->d,
                              reinterpret_cast<const __nv_bfloat16*>(L.wg.p), c->E, c->n_pred, c->k, c->ids.p,
                              c->wts.p, c->counts.p, c->block_counts.p, pred_counts, c->gate_partial.p, s));
  });
}

int moe_layer_forward(moe_ctx* c, int layer, const uint16_t* x, int T, uint16_t* y, int plan_mode, long iteration,
                      moe_layer_stats* stats, void* stream) {
  return guarded([&] {
    // a rank with no tokens still takes part in the exchange (x, y may be null)
    require(c && (T == 0 || (x && y)), "null argument");
    forward_device(c, layer, x, T, y, plan_mode, iteration, stats, pick(c, stream));
  });
}

int moe_layer_forward_host(moe_ctx* c, int layer, const uint16_t* x_host, int T, uint16_t* y_host, int plan_mode,
                           long iteration, moe_layer_stats* stats) {
  return guarded([&] {
    require(c && x_host && y_host, "null argument");
    require(T >= 0 && T <= c->Tmax, "token count exceeds max_tokens");
    if (!c->x_in.p) {
      c->x_in.alloc(static_cast<size_t>(c->Tmax) * c->xw);
      c->y_out.alloc(static_cast<size_t>(c->Tmax) * c->xw);
    }
    const size_t bytes = static_cast<size_t>(T) * c->xw * 2;
    CU_CHECK(cudaMemcpyAsync(c->x_in.p, x_host, bytes, cudaMemcpyHostToDevice, c->stream));
    forward_device(c, layer, c->x_in.p, T, c->y_out.p, plan_mode, iteration, stats, c->stream);
    CU_CHECK(cudaMemcpyAsync(y_host, c->y_out.p, bytes, cudaMemcpyDeviceToHost, c->stream));
    CU_CHECK(cudaStreamSynchronize(c->stream));
  });
}

int moe_layer_forward_host_async(moe_ctx* c, int layer, const uint16_t* x_host, int T, uint16_t* y_host,
                                 int plan_mode, long iteration, int64_t* ticket) {
  return guarded([&] {
    require(c && x_host && y_host, "null argument");
    require(T >= 0 && T <= c->Tmax, "token count exceeds max_tokens");
    if (!c->h2d) {
      CU_CHECK(cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking));
      CU_CHECK(cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking));
      for (int i = 0; i < 2; ++i) {
        c->xa[i].alloc(static_cast<size_t>(c->Tmax) * c->xw);
        c->ya[i].alloc(static_cast<size_t>(c->Tmax) * c->xw);
        for (cudaEvent_t* e : {&c->ev_x_ready[i], &c->ev_x_free[i], &c->ev_y_ready[i], &c->ev_done[i]}) {
          CU_CHECK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
          CU_CHECK(cudaEventRecord(*e, c->stream));  // "already satisfied" for the first use
        }
      }
      for (cudaEvent_t& e : c->ev_ticket) CU_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    const int64_t tk = c->next_ticket++;
    const int slot = static_cast<int>(tk & 1);
    const size_t bytes = static_cast<size_t>(T) * c->xw * 2;
    // upload: wait until the call two steps back has finished reading this slot
    CU_CHECK(cudaStreamWaitEvent(c->h2d, c->ev_x_free[slot], 0));
    CU_CHECK(cudaMemcpyAsync(c->xa[slot].p, x_host, bytes, cudaMemcpyHostToDevice, c->h2d));
    CU_CHECK(cudaEventRecord(c->ev_x_ready[slot], c->h2d));
    // compute: this slot's output buffer must have been downloaded (call tk-2)
    CU_CHECK(cudaStreamWaitEvent(c->stream, c->ev_x_ready[slot], 0));
    CU_CHECK(cudaStreamWaitEvent(c->stream, c->ev_done[slot], 0));
    forward_device(c, layer, c->xa[slot].p, T, c->ya[slot].p, plan_mode, iteration, nullptr, c->stream,
                   c->ev_x_free[slot]);
    CU_CHECK(cudaEventRecord(c->ev_y_ready[slot], c->stream));
    // download on its own stream so it overlaps the next step's layer
    CU_CHECK(cudaStreamWaitEvent(c->d2h, c->ev_y_ready[slot], 0));
    CU_CHECK(cudaMemcpyAsync(y_host, c->ya[slot].p, bytes, cudaMemcpyDeviceToHost, c->d2h));
    CU_CHECK(cudaEventRecord(c->ev_done[slot], c->d2h));
    CU_CHECK(cudaEventRecord(c->ev_ticket[tk % moe_ctx::kTicketRing], c->d2h));
    if (ticket) *ticket = tk;
  });
}

int moe_residency(moe_ctx* c, int layer, int32_t* slot_of, int* n_slots) {
  return guarded([&] {
    Layer& L = layer_at(c, layer);
    require(slot_of != nullptr, "null argument");
    if (c->placed) {
      ensure_pools(c, L);
      for (int e = 0; e < c->E; ++e) slot_of[e] = L.slot_of[e];
    } else {
      for (int e = 0; e < c->E; ++e) slot_of[e] = e;
    }
    if (n_slots) *n_slots = c->placed ? c->slots : c->E;
  });
}

int moe_gemm_times(moe_ctx* c, int max_n, float* g1, float* g2, int64_t* rows, int* n_out) {
  return guarded([&] {
    require(c && n_out, "null argument");
    CU_CHECK(cudaStreamSynchronize(c->stream));
    const int64_t avail = std::min<int64_t>(c->gemm_seq, moe_ctx::kGemmRing);
    const int n = static_cast<int>(std::min<int64_t>(avail, std::max(0, max_n)));
    for (int i = 0; i < n; ++i) {
      const int slot = static_cast<int>((c->gemm_seq - n + i) % moe_ctx::kGemmRing);
      float a = 0.0f, b = 0.0f;
      if (c->use_pdl) {  // GEMM1 and GEMM2 overlap: one interval
        CU_CHECK(cudaEventElapsedTime(&a, c->gemm_ev[slot][0], c->gemm_ev[slot][2]));
      } else {
        CU_CHECK(cudaEventElapsedTime(&a, c->gemm_ev[slot][0], c->gemm_ev[slot][1]));
        CU_CHECK(cudaEventElapsedTime(&b, c->gemm_ev[slot][1], c->gemm_ev[slot][2]));
      }
      if (g1) g1[i] = a;
      if (g2) g2[i] = b;
      if (rows) rows[i] = c->gemm_rows[slot];
    }
    *n_out = n;
  });
}

int moe_host_alloc(size_t bytes, void** out) {
  return guarded([&] {
    require(out != nullptr, "null argument");
    CU_CHECK(cudaHostAlloc(out, bytes, cudaHostAllocPortable | cudaHostAllocMapped));
  });
}

int moe_host_free(void* p) {
  return guarded([&] {
    if (p) CU_CHECK(cudaFreeHost(p));
  });
}

int moe_wait(moe_ctx* c, int64_t ticket) {
  return guarded([&] {
    require(c != nullptr, "null context");
    require(ticket >= 0 && ticket < c->next_ticket, "unknown ticket");
    // this call's own completion event (a ticket more than kTicketRing calls old
    // shares its event with a later call, which completes later: conservative)
    CU_CHECK(cudaEventSynchronize(c->ev_ticket[ticket % moe_ctx::kTicketRing]));
    flush_pending_plan(c);
  });
}

int moe_forward_begin(moe_ctx* c, int layer, const uint16_t* x, int T, const int32_t* counts_all, void* stream) {
  return guarded([&] {
    Layer& L = layer_at(c, layer);
    require(x != nullptr, "null input");
    require(T >= 0 && T <= c->Tmax, "token count exceeds max_tokens");
    require(!c->p2p, "the staged API is for the NCCL / external exchange, not MOE_EXCHANGE_P2P");
    cudaStream_t s = pick(c, stream);
    flush_pending_plan(c);
    if (!counts_all) {
      // stage 1: gate only; caller reads counts (moe_buffer 7), all-gathers, calls again
      stage_gate(c, L, x, T, s, nullptr);
      CU_CHECK(cudaStreamSynchronize(s));
      c->cur_layer = layer;
      c->cur_T = T;
      c->cur_x = x;
      return;
    }
    require(c->cur_layer == layer && c->cur_x == x && c->cur_T == T, "forward_begin stage 2 without stage 1");
    stage_plan(c, layer, MOE_PLAN_FIXED, 0, counts_all, c->E);
    stage_dispatch(c, x, T, s);
    CU_CHECK(cudaStreamSynchronize(s));
  });
}

int moe_forward_expert(moe_ctx* c, int layer, void* stream) {
  return guarded([&] {
    layer_at(c, layer);
    require(c->cur_layer == layer, "forward_expert without forward_begin");
    stage_expert(c, layer, pick(c, stream));
    CU_CHECK(cudaStreamSynchronize(pick(c, stream)));
  });
}

int moe_forward_end(moe_ctx* c, uint16_t* y, void* stream) {
  return guarded([&] {
    require(c && y, "null argument");
    require(c->cur_layer >= 0, "forward_end without forward_begin");
    stage_combine(c, y, c->cur_T, pick(c, stream));
    CU_CHECK(cudaStreamSynchronize(pick(c, stream)));
    c->cur_layer = -1;
  });
}

int moe_buffer(moe_ctx* c, int which, void** ptr, int64_t* rows) {
  return guarded([&] {
    require(c && ptr, "null argument");
    flush_pending_plan(c);
    int64_t r = 0;
    switch (which) {
      case 0: *ptr = c->xp.p; r = c->plan.rows_local; break;
      case 1: *ptr = c->send.p; r = c->plan.rows_send; break;
      case 2: *ptr = c->yp.p; r = c->plan.rows_local; break;
      case 3: *ptr = c->ret.p; r = c->plan.rows_send; break;
      case 4: *ptr = c->ids.p; r = static_cast<int64_t>(c->cur_T) * c->k; break;
      case 5: *ptr = c->wts.p; r = static_cast<int64_t>(c->cur_T) * c->k; break;
      case 6: *ptr = c->row_code.p; r = static_cast<int64_t>(c->cur_T) * c->k; break;
      case 7: *ptr = c->counts.p; r = c->E; break;
      case 8: *ptr = c->h.p; r = c->plan.rows_local; break;
      case 9: *ptr = c->p2p ? c->slab.p + c->off_flags : nullptr; r = kFlagKinds * kMaxRanks; break;  // P2P flags
      case 10: *ptr = c->epoch_dev.p; r = 1; break;  // P2P device epoch
      case 11: *ptr = c->perm_src.p; r = c->plan.rows_local; break;  // gathered GEMM1: row -> token
      default: throw std::invalid_argument("unknown buffer id");
    }
    if (rows) *rows = r;
  });
}

int moe_memcpy(moe_ctx* c, void* dst, const void* src, size_t bytes) {
  return guarded([&] {
    require(c && dst && src, "null argument");
    CU_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, c->stream));
    CU_CHECK(cudaStreamSynchronize(c->stream));
  });
}

int moe_exchange_plan(int G, int rank, int E, const int32_t* counts_all, const int32_t* rc, const int32_t* rg,
                      moe_chunk* sends, int* n_sends, moe_chunk* recvs, int* n_recvs, int max_chunks,
                      int64_t* rows_local, int64_t* rows_send, int64_t* seg_start, int64_t* seg_rows) {
  return guarded([&] {
    require(counts_all && rc && rg, "null argument");
    std::vector<int64_t> all(static_cast<size_t>(G) * std::max(E, 0));
    for (size_t i = 0; i < all.size(); ++i) all[i] = counts_all[i];
    HostPlan hp;
    build_exchange_plan(G, rank, E, all.data(), rc, rg, hp);
    require(static_cast<int>(hp.sends.size()) <= max_chunks && static_cast<int>(hp.recvs.size()) <= max_chunks,
            "chunk arrays too small");
    auto copy = [](const std::vector<Chunk>& v, moe_chunk* dst) {
      for (size_t i = 0; i < v.size(); ++i) dst[i] = moe_chunk{v[i].peer, v[i].replica, v[i].row_offset, v[i].rows};
    };
    if (sends) copy(hp.sends, sends);
    if (recvs) copy(hp.recvs, recvs);
    if (n_sends) *n_sends = static_cast<int>(hp.sends.size());
    if (n_recvs) *n_recvs = static_cast<int>(hp.recvs.size());
    if (rows_local) *rows_local = hp.rows_local;
    if (rows_send) *rows_send = hp.rows_send;
    for (int i = 0; i < hp.dev.R; ++i) {
      if (seg_start) seg_start[i] = hp.seg_start[i];
      if (seg_rows) seg_rows[i] = hp.rep_size[i];
    }
  });
}

int moe_exchange_plan_direct(int G, int rank, int E, const int32_t* counts_all, const int32_t* rc, const int32_t* rg,
                             int32_t* rep_target, int32_t* rep_row_base, int64_t* rows_local, int64_t* rows_send) {
  return guarded([&] {
    require(counts_all && rc && rg, "null argument");
    std::vector<int64_t> all(static_cast<size_t>(G) * std::max(E, 0));
    for (size_t i = 0; i < all.size(); ++i) all[i] = counts_all[i];
    HostPlan hp;
    build_exchange_plan(G, rank, E, all.data(), rc, rg, hp, /*direct=*/true);
    for (int f = 0; f < hp.dev.R; ++f) {
      if (rep_target) rep_target[f] = hp.dev.rep_remote[f];
      if (rep_row_base) rep_row_base[f] = hp.dev.rep_row_base[f];
    }
    if (rows_local) *rows_local = hp.rows_local;
    if (rows_send) *rows_send = hp.rows_send;
  });
}

// ------------------------------------------------------------- planner API
int moe_plan_scale(const int64_t* loads, int E, int layer, double mem, double cap, double cv, int excl,
                   int32_t* counts_out, double* alloc_out, int* steps_out, int32_t* split, double* cvt, int cap_n) {
  return guarded([&] {
    require(loads && counts_out, "null argument");
    moeless::ModelSpec m;
    m.experts_per_layer = E;
    m.top_k = 1;
    m.expert_mem_mb = mem;
    m.layer_mem_cap_mb = cap;
    moeless::ScalerConfig sc;
    sc.cv_threshold = cv;
    sc.exclude_zero_loads_from_cv = excl != 0;
    moeless::ScaleTrace tr;
    moeless::LoadVector lv{layer, std::vector<int64_t>(loads, loads + std::max(E, 0))};
    auto plan = moeless::scale_experts(lv, m, sc, &tr);
    std::copy(plan.replica_counts.begin(), plan.replica_counts.end(), counts_out);
    if (alloc_out) *alloc_out = plan.alloc_mem_mb;
    if (steps_out) *steps_out = static_cast<int>(tr.split_expert.size());
    for (int i = 0; i < cap_n && i < static_cast<int>(tr.split_expert.size()); ++i) {
      if (split) split[i] = tr.split_expert[i];
      if (cvt) cvt[i] = tr.cv[i];
    }
  });
}

struct moe_registry {
  moeless::ReplicaRegistry reg;
};

int moe_registry_create(int keep_alive, moe_registry** out) {
  return guarded([&] {
    require(out != nullptr, "null argument");
    *out = new moe_registry{moeless::ReplicaRegistry(keep_alive)};
  });
}
int moe_registry_destroy(moe_registry* r) {
  delete r;
  return MOE_OK;
}
int64_t moe_registry_size(const moe_registry* r) { return r ? static_cast<int64_t>(r->reg.size()) : -1; }

namespace {
moeless::ScalingPlan plan_of(const int64_t* loads, const int32_t* counts, int E, int layer, double mem) {
  moeless::ScalingPlan p;
  p.layer = layer;
  p.expert_mem_mb = mem;
  p.replica_counts.assign(counts, counts + E);
  int extra = 0;
  for (int e = 0; e < E; ++e) {
    extra += counts[e] - 1;
    for (int r = 0; r < counts[e]; ++r) p.shares.push_back({e, r, moeless::Rational(loads[e], counts[e])});
  }
  p.alloc_mem_mb = extra * mem;
  return p;
}
moeless::Placement placement_of(const int32_t* counts, const int32_t* gpu, int E, int G, int layer, double mem) {
  moeless::Placement p;
  p.layer = layer;
  p.per_gpu_mem_mb.assign(G, 0.0);
  int i = 0;
  for (int e = 0; e < E; ++e) {
    p.gpu_for.emplace_back();
    for (int r = 0; r < counts[e]; ++r, ++i) {
      p.gpu_for.back().push_back(gpu[i]);
      if (gpu[i] >= 0 && gpu[i] < G) p.per_gpu_mem_mb[gpu[i]] += mem;
    }
  }
  return p;
}
}  // namespace

int moe_plan_place(moe_registry* r, const int64_t* loads, const int32_t* counts, int E, int layer, double mem, int G,
                   double cap, long it, int incl, double alpha, double beta, int32_t* gpu_out, int* warm, int* cold) {
  return guarded([&] {
    require(r && loads && counts && gpu_out, "null argument");
    for (int e = 0; e < E; ++e) require(counts[e] >= 1, "replica count must be >= 1");
    auto plan = plan_of(loads, counts, E, layer, mem);
    moeless::ClusterSpec cl;
    cl.gpu_count = G;
    cl.gpu_mem_capacity_mb = cap;
    moeless::PlacerOptions opt;
    opt.load_includes_compute = incl != 0;
    opt.alpha_ms_per_token = alpha;
    opt.beta_ms_per_token = beta;
    auto res = moeless::place_experts(plan, cl, r->reg, it, opt);
    int i = 0;
    for (int e = 0; e < E; ++e)
      for (int g : res.placement.gpu_for[e]) gpu_out[i++] = g;
    if (warm) *warm = res.warm_count;
    if (cold) *cold = res.cold_count;
  });
}

int moe_registry_update(moe_registry* r, const int32_t* counts, const int32_t* gpu, int E, int G, int layer, long it) {
  return guarded([&] {
    require(r && counts && gpu, "null argument");
    moeless::update_registry(r->reg, placement_of(counts, gpu, E, G, layer, 1.0), it);
  });
}

int moe_model_forward_time(const int64_t* loads, const int32_t* counts, const int32_t* gpu, const int64_t* actual,
                           int E, int G, double alpha, double beta, double t_misc, double m_misc, double mem,
                           double* out6) {
  return guarded([&] {
    require(loads && counts && gpu && actual && out6, "null argument");
    auto plan = plan_of(loads, counts, E, 0, mem);
    auto pl = placement_of(counts, gpu, E, G, 0, mem);
    moeless::ClusterSpec cl;
    cl.gpu_count = G;
    cl.alpha_ms_per_token = alpha;
    cl.beta_ms_per_token = beta;
    cl.t_misc_ms = t_misc;
    cl.m_misc_mb = m_misc;
    moeless::ModelSpec ms;
    ms.experts_per_layer = E;
    ms.expert_mem_mb = mem;
    auto m = moeless::layer_forward_time(plan, pl, moeless::LoadVector{0, std::vector<int64_t>(actual, actual + E)}, cl,
                                         ms);
    out6[0] = m.compute_ms;
    out6[1] = m.comm_ms;
    out6[2] = m.forward_ms;
    out6[3] = m.replica_count;
    out6[4] = m.mem_mb;
    out6[5] = m.cost_mb_ms;
  });
}

int moe_plan_predict(int kind, const int64_t* actual, int E, int layer, const int64_t* history, int hlen,
                     const double* acc, int L, int distance, double decay, int window, long it, uint64_t seed,
                     const double* pop, int64_t* out, int* fallback) {
  return guarded([&] {
    require(actual && out, "null argument");
    require(kind >= 0 && kind <= 2, "unknown predictor kind");
    moeless::PredictorProfile p;
    p.kind = static_cast<moeless::PredictorKind>(kind);
    p.distance = distance;
    p.distance_decay = decay;
    p.history_window = window;
    if (acc) p.per_layer_accuracy.assign(acc, acc + L);
    std::vector<moeless::LoadVector> hist;
    for (int i = 0; i < hlen; ++i)
      hist.push_back({layer, std::vector<int64_t>(history + static_cast<size_t>(i) * E, history + static_cast<size_t>(i + 1) * E)});
    std::vector<double> pw;
    if (pop) pw.assign(pop, pop + E);
    bool fb = false;
    auto r = moeless::predict({layer, std::vector<int64_t>(actual, actual + E)}, hist, p, it, seed, pw, &fb);
    std::copy(r.loads.begin(), r.loads.end(), out);
    if (fallback) *fallback = fb ? 1 : 0;
  });
}

double moe_measure_accuracy(const int64_t* pred, const int64_t* actual, int E) {
  double v = -1.0;
  int rc = guarded([&] {
    v = moeless::measure_accuracy({0, std::vector<int64_t>(pred, pred + E)}, {0, std::vector<int64_t>(actual, actual + E)});
  });
  return rc == MOE_OK ? v : -1.0;
}

double moe_percentile(const double* v, int n, double q) {
  double out = -1.0;
  int rc = guarded([&] { out = moeless::percentile(std::vector<double>(v, v + std::max(n, 0)), q); });
  return rc == MOE_OK ? out : -1.0;
}

int moe_route_tokens(int64_t T, int layer, long it, int E, int L, double s, uint64_t seed, int k, int drift,
                     int64_t* loads) {
  return guarded([&] {
    require(loads != nullptr, "null argument");
    auto prof = moeless::make_popularity_profile(E, L, s, seed, false, drift);
    moeless::IterationBatch b;
    b.iteration = it;
    b.token_count = T;
    auto lv = moeless::route_tokens(b, layer, prof, k, E, seed);
    std::copy(lv.loads.begin(), lv.loads.end(), loads);
  });
}

int moe_popularity(int E, int L, double s, uint64_t seed, int layer, long it, int drift, int32_t* perm, double* w) {
  return guarded([&] {
    auto prof = moeless::make_popularity_profile(E, L, s, seed, false, drift);
    auto p = moeless::effective_permutation(prof, layer, it);
    if (perm) std::copy(p.begin(), p.end(), perm);
    if (w) {
      auto ww = moeless::popularity_weights(prof, layer, it, moeless::Phase::prefill);
      std::copy(ww.begin(), ww.end(), w);
    }
  });
}

uint64_t moe_stream_key(uint64_t seed, uint64_t a, uint64_t b, uint64_t tag) { return stream_key(seed, a, b, tag); }

int moe_synth_tokens(uint64_t key, int64_t first, int64_t T, int d, int E, uint16_t* x) {
  return guarded([&] {
    require(x && T >= 0 && d > E && E >= 1, "bad synth_tokens arguments");
    synth_tokens(key, first, T, d, E, x);
  });
}

int moe_synth_gate(uint64_t key, int d, int E, const double* pop, const int32_t* noise_perm, uint16_t* wg) {
  return guarded([&] {
    require(pop && noise_perm && wg && d > E, "bad synth_gate arguments");
    synth_gate(key, d, E, pop, noise_perm, wg);
  });
}

int moe_synth_expert(uint64_t key, int d, int ff, uint16_t* w1, uint16_t* w3, uint16_t* w2) {
  return guarded([&] {
    require(w1 && w3 && w2, "null argument");
    synth_expert(key, d, ff, w1, w3, w2);
  });
}

}  // extern "C"
