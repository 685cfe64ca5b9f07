/*
 * moe_b200.h — C-ABI of the B200-native MoE-layer data path (drop-in boundary).
 *
 * The reference (MoEless, /root/reference) has no FFI: its boundary is the
 * value-semantic C++ API in proj/include/moeless/.  This header is the thin
 * C layer that API's callers reach the GPU through.  Every
 * entry point names the reference interface it replaces or serves:
 *
 *   moe_layer_forward / moe_layer_forward_host
 *       replaces LayerMetrics layer_forward_time(plan, placement, actual,
 *       cluster, model)            proj/include/moeless/cost_model.hpp:24-26
 *       (the analytic alpha*max_share + 2*beta*max_gpu + t_misc becomes a real
 *       gate -> dispatch -> SwiGLU FFN -> combine on tcgen05 tensor cores).
 *   moe_gate_topk
 *       replaces LoadVector route_tokens(...)   proj/include/moeless/workload.hpp:90-92
 *   moe_predict_loads
 *       serves LoadVector predict(...)          proj/include/moeless/predictor.hpp:40-43
 *       (a real gate-shaped predictor kernel)
 *   moe_set_placement
 *       consumes ScalingPlan.replica_counts     proj/include/moeless/types.hpp:59
 *       and Placement.gpu_for                   proj/include/moeless/placer.hpp:17
 *   moe_plan_scale / moe_plan_place / moe_registry_*
 *       scale_experts                           proj/include/moeless/scaler.hpp:29-30
 *       place_experts / update_registry         proj/include/moeless/placer.hpp:74-80
 *       (host C++; exported so non-C++ callers and the tests reach them too)
 *
 * Conventions
 *   - bf16 tensors are passed as uint16_t bit patterns, row-major.
 *   - Weights use the nn.Linear layout: W1, W3 [d_ff, d_model], W2 [d_model,
 *     d_ff], Wg [E, d_model].  FFN_e(x) = W2 (silu(W1 x) * (W3 x)).
 *   - Status codes: MOE_OK; MOE_EINVAL -> the C++ shim rethrows
 *     std::invalid_argument; MOE_EINFEASIBLE -> std::runtime_error (message
 *     keeps the reference wording, e.g. "no GPU has memory for replica (e,r)
 *     of layer l"); MOE_ECUDA / MOE_ENCCL -> std::runtime_error with the API
 *     error string.  No exception crosses this boundary; moe_last_error()
 *     returns the thread-local message of the last failure.
 *   - A context is single-threaded (one per host thread, mirroring
 *     run_comparison's one-run-per-thread model, simulator.cpp:303-307) and
 *     bound to one device = one rank.  Multi-GPU runs use one process per GPU;
 *     the ranks share an NCCL unique id passed in moe_ctx_desc.
 *   - Device-pointer entry points take a cudaStream_t as void*; NULL means the
 *     context's own stream.  There is no CPU fallback: without a usable sm_100
 *     device moe_ctx_create fails with MOE_ECUDA.
 */
#ifndef MOE_B200_H_
#define MOE_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  MOE_OK = 0,
  MOE_EINVAL = 1,
  MOE_EINFEASIBLE = 2,
  MOE_ECUDA = 3,
  MOE_ENCCL = 4,
  MOE_ESTATE = 5
};

/* exchange modes for world_size > 1.
   NCCL:     counts all-gather + grouped ncclSend/ncclRecv of row chunks.
   EXTERNAL: the staged API; the caller moves the chunks.
   P2P:      peer memory over NVLink (or ranks sharing one device): dispatch
             stores rows straight into the owning rank's receive buffer and
             combine reads expert outputs from the owner; flags in device
             memory order the phases.  Requires moe_p2p_export/import.
   COPY:     the NCCL path's chunked exchange (same chunk lists and message
             order) over a copy-engine transport for ranks of ONE process
             (threads; any devices, peers on one GPU included): a host
             rendezvous per step, then cudaMemcpyAsync pulls.  The group is
             the 128 bytes in nccl_unique_id (any value shared by the ranks).
             Built for multi-rank testing on one GPU and for a single process
             driving several GPUs. */
enum { MOE_EXCHANGE_NCCL = 0, MOE_EXCHANGE_EXTERNAL = 1, MOE_EXCHANGE_P2P = 2, MOE_EXCHANGE_COPY = 3 };

/* planning modes for moe_layer_forward */
enum {
  MOE_PLAN_FIXED = 0, /* use the placement last given to moe_set_placement            */
  MOE_PLAN_SYNC = 1,  /* scale_experts + place_experts on this layer's actual counts
                         (oracle predictor, distance 0) inside the forward           */
  MOE_PLAN_PREDICTED = 2 /* MoEless: the fused predictor at layer l scores layer
                         l + predictor_distance; the host plans that layer from the
                         prediction ahead of time; layers never predicted (l < d)
                         bootstrap from their load history (simulator.cpp:146-151) */
};

typedef struct moe_ctx moe_ctx;

typedef struct {
  int num_layers;
  int num_experts;      /* E  */
  int top_k;            /* k  */
  int d_model;          /* multiple of 256 */
  int d_ff;             /* multiple of 128 */
  int max_tokens;       /* per-rank token capacity of one forward */
  int world_size;       /* G (1 = single GPU) */
  int rank;
  int device;           /* CUDA ordinal */
  int exchange_mode;    /* MOE_EXCHANGE_* (ignored when world_size == 1) */
  const void* nccl_unique_id; /* 128 bytes, same on every rank; NULL if G == 1 or external */
  int num_predictor_targets;  /* n target layers the fused predictor scores (0 = off) */
  /* planner knobs used by MOE_PLAN_SYNC (ModelSpec / ScalerConfig / ClusterSpec) */
  double expert_mem_mb;
  double layer_mem_cap_mb;
  double gpu_mem_capacity_mb;
  double cv_threshold;
  int keep_alive_iters;
  int predictor_distance;     /* d: predictor slot 0 of layer l scores layer l + d (default 1) */
  int precision;              /* MOE_PRECISION_BF16 (default) or MOE_PRECISION_FP32 */
  int use_cuda_graphs;        /* 1: single-GPU forwards are captured once per (layer, tokens,
                                 buffers) and replayed as one CUDA graph launch */
  int residency;              /* MOE_RESIDENCY_ALL (default) or MOE_RESIDENCY_PLACED */
  int replica_slots;          /* PLACED: cache slots per layer for replicas of non-home experts
                                 (0 = min(E - home, gpu_mem_capacity_mb / expert_mem_mb)) */
  int reserved[2];
} moe_ctx_desc;

/* Expert weight residency (the reference's ReplicaRegistry
   keep-alive, proj/src/placer.cpp:11-43,124-130, and cold starts,
   simulator.cpp:198-199).
   ALL:    every expert of every layer is resident on every rank (180 GB of HBM
           holds a 32-layer Mixtral stack), so any placement runs without
           copies.
   PLACED: rank g permanently holds only its home experts (e mod G == g, the
           static_plan placement, baselines.cpp:32-60) plus replica_slots cache
           slots per layer.  When a placement puts a replica of a non-home
           expert on g and the expert is not cached, its weights are copied
           from the home rank's slot over NVLink (peer memory, copy engine, on
           a side stream ordered after the layer's previous forward) into a
           free or least-recently-used slot; the layer's GEMMs wait for the
           copy.  A placement planned d layers ahead (MOE_PLAN_PREDICTED)
           therefore pre-warms its replicas while the layers between run; a
           synchronous plan (MOE_PLAN_SYNC) pays the copy on the critical path
           — the measured cold start.  Requires MOE_EXCHANGE_P2P (G > 1); at
           G == 1 every expert is home.  moe_load_expert_weights stores home
           experts only (calls for other experts are accepted and ignored). */
enum { MOE_RESIDENCY_ALL = 0, MOE_RESIDENCY_PLACED = 1 };

/* precision of activations, weights and outputs.  BF16: bf16 in/out, fp32
   accumulate on tcgen05 (tolerance 2e-2).  FP32: fp32 in/out, fp32 FFMA
   (tolerance 1e-4); activation/output buffers are float, weights are loaded
   with the *_f32 entry points. */
enum { MOE_PRECISION_BF16 = 0, MOE_PRECISION_FP32 = 1 };

typedef struct {
  /* LayerMetrics-compatible fields (types.hpp:73-80), measured */
  double compute_ms;   /* grouped GEMMs (K4) */
  double comm_ms;      /* one direction of the expert all-to-all (mean of both) */
  double forward_ms;   /* gate -> combine, device time */
  int replica_count;
  double mem_mb;
  /* per-phase device times, ms */
  double gate_ms, plan_ms, dispatch_ms, a2a_dispatch_ms, gemm1_ms, gemm2_ms, a2a_combine_ms,
      combine_ms;
  int64_t rows_local;  /* rows this rank's GEMMs processed */
  int64_t rows_sent;
  int warm_count, cold_count;
  int32_t counts[256];          /* this rank's gate histogram (E <= 256) */
  double predictor_accuracy;    /* measure_accuracy(prediction made d layers ago, actual); -1 if none */
  int32_t plan_source;          /* 0 fixed, 1 actual loads, 2 predicted ahead, 3 history bootstrap */
  /* MOE_RESIDENCY_PLACED: weight movement caused by this layer's latest placement */
  int32_t weight_copies;        /* experts copied into cache slots (cold) */
  int32_t weight_hits;          /* non-home experts already cached (warm) */
  double weight_copy_ms;        /* copy-stream time of those copies (0 if none) */
  double weight_copy_mb;        /* bytes copied, MB */
} moe_layer_stats;

const char* moe_last_error(void);
const char* moe_version(void);

/* ---------------------------------------------------------------- context */
/* 128-byte NCCL unique id for moe_ctx_desc.nccl_unique_id (rank 0 creates it,
   the launcher broadcasts it). */
int moe_nccl_unique_id(void* out128);
int moe_ctx_create(const moe_ctx_desc* desc, moe_ctx** out);

/* Peer-memory exchange (MOE_EXCHANGE_P2P).  Each rank exports a handle to its
   exchange slab, the launcher all-gathers the handles (any transport: MPI,
   torch.distributed, a file), and every rank imports all G of them, indexed by
   rank.  Handles from the same process are used as plain device pointers
   (several ranks may share one device); others are opened with CUDA IPC.
   Every rank must then issue the same sequence of moe_layer_forward calls. */
typedef struct {
  unsigned char ipc[64]; /* cudaIpcMemHandle_t of the slab */
  uint64_t pid;          /* exporting process */
  uint64_t base;         /* slab address in the exporting process */
  uint64_t bytes;        /* slab size */
  uint64_t off_flags, off_counts, off_xp, off_yp;
  int32_t device, rank, world_size, version;
  uint64_t off_weights;  /* MOE_RESIDENCY_PLACED: weight slots inside the slab */
  uint64_t weight_bytes;
  unsigned char reserved[40];
} moe_p2p_handle;        /* 192 bytes */
int moe_p2p_export(moe_ctx* ctx, moe_p2p_handle* out);
int moe_p2p_import(moe_ctx* ctx, const moe_p2p_handle* handles, int n);
int moe_ctx_destroy(moe_ctx* ctx);
int moe_ctx_stream(moe_ctx* ctx, void** stream_out);
int moe_ctx_sync(moe_ctx* ctx);

/* ---------------------------------------------------------------- weights */
/* Host (pinned or pageable) bf16 arrays; copied into the ctx-owned pool.  */
int moe_load_expert_weights(moe_ctx* ctx, int layer, int expert, const uint16_t* w1,
                            const uint16_t* w3, const uint16_t* w2);
int moe_set_gate_weights(moe_ctx* ctx, int layer, const uint16_t* wg);
/* fp32-mode counterparts (MOE_PRECISION_FP32 contexts only) */
int moe_load_expert_weights_f32(moe_ctx* ctx, int layer, int expert, const float* w1, const float* w3,
                                const float* w2);
int moe_set_gate_weights_f32(moe_ctx* ctx, int layer, const float* wg);
/* Gate weights already in device memory ([E, d_model], the context's
   precision): a stream-ordered device-to-device copy (stream NULL = the
   context's), so per-call gate updates cost no host staging. */
int moe_set_gate_weights_device(moe_ctx* ctx, int layer, const void* wg_dev, void* stream);
/* predictor weights for target `slot` (< num_predictor_targets), scored from
   layer `layer`'s hidden states: [E, d_model] */
int moe_set_predictor_weights(moe_ctx* ctx, int layer, int slot, const uint16_t* wp);
/* The batched predictor MLP for target `slot`: hidden = relu(x W1^T) with
   E hidden units (W1 [E, d_model] bf16, computed in the gate's read of x),
   out[e] = sum_j W2[e][j] hidden[j] (W2 [E, E] fp32, accumulated in j order
   with fused multiply-adds), histogram of top-k(out).  w1 NULL keeps the
   slot's current rows; w2 NULL returns the slot to the linear predictor.
   The paper's predictor is a gate-shaped linear on layer-l hidden states
   (PAPER.md:469,696,1069); this slot type adds one hidden layer.  It serves
   the reference's predict() interface (predictor.hpp:40-43, dispatch at
   predictor.cpp:146-166), whose stand-ins predict_noisy / predict_historical
   (predictor.cpp:54-142) only perturb the answer key. */
int moe_set_predictor_mlp(moe_ctx* ctx, int layer, int slot, const uint16_t* w1, const float* w2);

/* ------------------------------------------------------------- placement */
/* replica_counts[E] >= 1; replica_gpu[sum R] flattened (expert, ordinal).   */
int moe_set_placement(moe_ctx* ctx, int layer, const int32_t* replica_counts,
                      const int32_t* replica_gpu);

/* The placement in force for `layer` (after the last forward's planning):
   replica_counts[E] and replica_gpu[*n_replicas] flattened (expert, ordinal),
   i.e. ScalingPlan.replica_counts / Placement.gpu_for (types.hpp:59,
   placer.hpp:17).  replica_gpu may be NULL to query the size. */
int moe_get_placement(moe_ctx* ctx, int layer, int32_t* replica_counts, int32_t* replica_gpu, int max_replicas,
                      int* n_replicas);

/* ---------------------------------------------------------- device kernels */
/* K1 (+K2): x_dev [T, d] -> ids [T, k], weights [T, k], counts [E] (zeroed
   internally).  pred_counts [n_pred, E] may be NULL. */
int moe_gate_topk(moe_ctx* ctx, int layer, const uint16_t* x_dev, int tokens, int32_t* ids_dev,
                  float* weights_dev, int32_t* counts_dev, int32_t* pred_counts_dev, void* stream);

/* K2 alone: per-target histograms of the predictor gates on x_dev. */
int moe_predict_loads(moe_ctx* ctx, int layer, const uint16_t* x_dev, int tokens,
                      int32_t* pred_counts_dev, void* stream);

/* Full layer: y_dev [T, d] = sum_j w_tj FFN_{e_tj}(x_t).  stats may be NULL. */
int moe_layer_forward(moe_ctx* ctx, int layer, const uint16_t* x_dev, int tokens, uint16_t* y_dev,
                      int plan_mode, long iteration, moe_layer_stats* stats, void* stream);

/* Several forwards as ONE CUDA graph (a decode step over many layers pays one
   graph launch, not one per layer): moe_graph_begin starts capturing the
   context's stream; the moe_layer_forward calls that follow (stream NULL,
   stats NULL, device-planned: G == 1, or FIXED / PREDICTED-ahead at G > 1;
   not with MOE_RESIDENCY_PLACED) are recorded instead of run; moe_graph_end
   instantiates them and returns *graph_id.  moe_graph_launch replays the
   graph on `stream` (NULL: the context's stream), ordered after the
   context's uploads.  Replays re-read each layer's current gate weights and
   inputs but do not run the host planner's per-forward bookkeeping (the
   device plans every layer).  Graphs are freed by moe_destroy. */
int moe_graph_begin(moe_ctx* ctx);
int moe_graph_end(moe_ctx* ctx, int* graph_id);
int moe_graph_launch(moe_ctx* ctx, int graph_id, void* stream);

/* The layer on caller-given routing (the SURVEY §8 c3 bridge): ids_dev [T, k]
   int32 expert ids and weights_dev [T, k] fp32 (NULL: 1/k each) replace K1, so
   routing produced outside the gate — e.g. the reference's route_tokens stream
   (proj/src/workload.cpp:188-230) replayed per token — drives K3 -> K4 -> K5
   unchanged and the load counts the planner sees are exactly the histogram of
   those ids.  A token must name k distinct experts in [0, E): otherwise
   MOE_EINVAL (returned by this call when stats != NULL, else by the next call
   that synchronises the context), that token's output being 0.  No predictor
   runs on this path. */
int moe_layer_forward_ids(moe_ctx* ctx, int layer, const uint16_t* x_dev, const int32_t* ids_dev,
                          const float* weights_dev, int tokens, uint16_t* y_dev, int plan_mode, long iteration,
                          moe_layer_stats* stats, void* stream);

/* The dispatch plan the device used for the most recent forward (synchronises
   the context): n_e[E] = assignments of expert e over all ranks; segs[3 * i ..]
   = (first row, rows, weight slot) of GEMM segment i on this rank (one per
   replica here with rows > 0; co-located replicas of an expert form one
   segment on a single GPU); *nseg segments; *rows_local their total. */
int moe_last_plan(moe_ctx* ctx, int32_t* n_e, int32_t* segs, int max_segs, int* nseg, int64_t* rows_local);

/* Same with HOST buffers: H2D of x and D2H of y happen inside (the e2e path). */
int moe_layer_forward_host(moe_ctx* ctx, int layer, const uint16_t* x_host, int tokens,
                           uint16_t* y_host, int plan_mode, long iteration,
                           moe_layer_stats* stats);

/* Pipelined host-buffer forward for serving loops: enqueues H2D(x) on a copy
   stream, the layer on the compute stream and D2H(y) on a second copy stream,
   and returns once the layer's device work is enqueued (it blocks only while
   the host planner waits for this step's gate histogram).  Consecutive calls
   therefore overlap step i+1's upload and step i-1's download with step i's
   GEMMs.  x_host/y_host must be pinned and stay valid until moe_wait(ticket)
   returns.  At most 2 calls may be in flight; *ticket identifies the call. */
int moe_layer_forward_host_async(moe_ctx* ctx, int layer, const uint16_t* x_host, int tokens,
                                 uint16_t* y_host, int plan_mode, long iteration,
                                 int64_t* ticket);
int moe_wait(moe_ctx* ctx, int64_t ticket);
/* K4 device times of the most recent forwards (<= 64), oldest first, measured
   with CUDA events recorded around the two grouped GEMMs of EVERY forward
   (no host synchronisation inside the forward).  Synchronises the ctx
   stream, then fills up to max_n entries and *n_out.  GEMM2 is launched
   programmatically behind GEMM1 (it streams its weights during GEMM1's
   tail), so by default gemm1_ms holds the GEMM1+GEMM2 interval and gemm2_ms
   is 0; env MOE_PDL=0 serialises them and reports them apart. */
int moe_gemm_times(moe_ctx* ctx, int max_n, float* gemm1_ms, float* gemm2_ms, int64_t* rows, int* n_out);

/* Page-locked host buffers for the pipelined API (portable + mapped). */
int moe_host_alloc(size_t bytes, void** out);
int moe_host_free(void* p);

/* Staged forward for MOE_EXCHANGE_EXTERNAL (tests / custom transports):
   begin = gate + plan + dispatch; expert = both GEMMs over the received rows;
   end = combine.  Between the stages the caller moves rows between ranks
   using the buffers and chunk tables below. */
int moe_forward_begin(moe_ctx* ctx, int layer, const uint16_t* x_dev, int tokens,
                      const int32_t* counts_all /* [G][E] host, NULL => local only */,
                      void* stream);
int moe_forward_expert(moe_ctx* ctx, int layer, void* stream);
int moe_forward_end(moe_ctx* ctx, uint16_t* y_dev, void* stream);
/* Device buffers of the staged forward: which = 0 recv/permuted X, 1 send X,
   2 expert output Y (recv layout), 3 return buffer (send layout), 4 ids,
   5 weights, 6 row codes, 7 counts, 8 SwiGLU intermediate H, 9 peer-exchange
   flags [4][8] u32 (P2P), 10 the P2P device epoch, 11 the row -> token list
   of a single-GPU forward whose GEMM1 gathers x in place (int32, written
   instead of buffer 0 there).  rows_out = valid rows. */
int moe_buffer(moe_ctx* ctx, int which, void** ptr_out, int64_t* rows_out);
/* Weight residency of one layer on this rank: slot_of[E] = weight slot the
   GEMMs read for expert e (-1: not resident here; ALL: slot_of[e] == e),
   n_slots_out = slots in the layer's pool. */
int moe_residency(moe_ctx* ctx, int layer, int32_t* slot_of, int* n_slots_out);
/* cudaMemcpyDefault-style copy between any host/device pointers (UVA), on the
   ctx stream, synchronous on return — the transport hook of the staged API. */
int moe_memcpy(moe_ctx* ctx, void* dst, const void* src, size_t bytes);

/* ------------------------------------------------ exchange plan (host C++) */
/* The integer replica split and the row exchange it implies, computed from
   every rank's gate histogram counts_all[G][E].  Chunks: {peer, replica,
   row_offset, rows}: sends are offsets into this rank's send buffer, recvs are
   offsets into its received-rows buffer.  Returns counts through *_n; arrays
   must hold sum R entries per peer (max_chunks total). */
typedef struct {
  int32_t peer;
  int32_t replica;
  int64_t row_offset;
  int64_t rows;
} moe_chunk;

int moe_exchange_plan(int world_size, int rank, int num_experts, const int32_t* counts_all,
                      const int32_t* replica_counts, const int32_t* replica_gpu,
                      moe_chunk* sends, int* n_sends, moe_chunk* recvs, int* n_recvs,
                      int max_chunks, int64_t* rows_local, int64_t* rows_send,
                      int64_t* seg_start /* [sum R], -1 if not local */,
                      int64_t* seg_rows /* [sum R] */);

/* The peer-memory (MOE_EXCHANGE_P2P) form of the same plan: for every replica
   f (flattened (expert, ordinal)), the rank whose received-rows buffer holds
   its rows (rep_target[f] == replica_gpu[f]) and rep_row_base[f] such that the
   assignment with global rank gr of the expert lands in row
   rep_row_base[f] + gr of that rank's buffer. */
int moe_exchange_plan_direct(int world_size, int rank, int num_experts, const int32_t* counts_all,
                             const int32_t* replica_counts, const int32_t* replica_gpu, int32_t* rep_target,
                             int32_t* rep_row_base, int64_t* rows_local, int64_t* rows_send);

/* ------------------------------------------------------- planner (host C++) */
/* scale_experts (scaler.hpp:29-30): counts_out[E]; trace arrays may be NULL. */
int moe_plan_scale(const int64_t* loads, int num_experts, int layer, double expert_mem_mb,
                   double layer_mem_cap_mb, double cv_threshold, int exclude_zero,
                   int32_t* counts_out, double* alloc_mem_out, int* steps_out,
                   int32_t* split_trace, double* cv_trace, int trace_cap);

typedef struct moe_registry moe_registry;
int moe_registry_create(int keep_alive_iters, moe_registry** out);
int moe_registry_destroy(moe_registry* reg);
int64_t moe_registry_size(const moe_registry* reg);

/* place_experts (placer.hpp:74-76) on a plan whose shares are plan_loads[e] /
   counts[e]; gpu_out[sum R] flattened (expert, ordinal). */
int moe_plan_place(moe_registry* reg, const int64_t* plan_loads, const int32_t* counts,
                   int num_experts, int layer, double expert_mem_mb, int gpus,
                   double gpu_mem_capacity_mb, long iteration, int load_includes_compute,
                   double alpha_ms_per_token, double beta_ms_per_token, int32_t* gpu_out,
                   int* warm_out, int* cold_out);
/* update_registry (placer.hpp:80) */
int moe_registry_update(moe_registry* reg, const int32_t* counts, const int32_t* gpu_flat,
                        int num_experts, int gpus, int layer, long iteration);

/* layer_forward_time (cost_model.hpp:24-26), the analytic model, for
   calibration: out6 = compute, comm, forward, replicas, mem, cost */
int moe_model_forward_time(const int64_t* plan_loads, const int32_t* counts,
                           const int32_t* gpu_flat, const int64_t* actual, int num_experts,
                           int gpus, double alpha, double beta, double t_misc, double m_misc,
                           double expert_mem_mb, double* out6);

/* predict (predictor.hpp:40-43): kind 0 oracle, 1 noisy, 2 historical. */
int moe_plan_predict(int kind, const int64_t* actual, int num_experts, int layer,
                     const int64_t* history, int history_len, const double* accuracy,
                     int num_layers, int distance, double decay, int window, long iteration,
                     uint64_t seed, const double* popularity, int64_t* out, int* fallback);
double moe_measure_accuracy(const int64_t* predicted, const int64_t* actual, int num_experts);
double moe_percentile(const double* values, int n, double q);

/* static_plan (baselines.cpp:32-60): expert e -> GPU e mod G, one replica
   each; gpu_out[E].  Throws the reference's "static placement does not fit
   GPU g" as MOE_EINFEASIBLE. */
int moe_static_plan(const int64_t* loads, int num_experts, int gpus, double expert_mem_mb,
                    double gpu_mem_capacity_mb, int32_t* gpu_out);
/* round_robin_placement (simulator.cpp:32-50): replica f (flattened
   (expert, ordinal)) -> GPU f mod G; gpu_out[sum counts]. */
int moe_round_robin_placement(const int32_t* counts, int num_experts, int gpus, double expert_mem_mb,
                              double gpu_mem_capacity_mb, int32_t* gpu_out);
/* gpu_comm_times (cost_model.cpp:67-89): beta x the shares hosted per GPU;
   out[G].  Shares are plan_loads[e] / counts[e]. */
int moe_gpu_comm_times(const int64_t* plan_loads, const int32_t* counts, const int32_t* gpu_flat,
                       int num_experts, int gpus, double beta_ms_per_token, double* out);
/* oracle_balance_time (baselines.cpp:141-154): the perfect-balance line;
   out6 = compute, comm, forward, replicas, mem, cost (as moe_model_forward_time). */
int moe_oracle_balance_time(const int64_t* actual, int num_experts, int gpus, double alpha, double beta,
                            double t_misc, double m_misc, double expert_mem_mb, double* out6);
/* verify_plan (scaler.cpp:99-173) on an explicit plan: replica counts[n_counts]
   and shares (expert, ordinal, num/den)[n_shares]; *ok and the reference's
   issue messages, newline-separated, in issues[cap]. */
int moe_verify_plan(const int64_t* loads, int num_experts, const int32_t* counts, int n_counts,
                    const int32_t* share_expert, const int32_t* share_ordinal, const int64_t* share_num,
                    const int64_t* share_den, int n_shares, double alloc_mem_mb, double expert_mem_mb,
                    double layer_mem_cap_mb, double cv_threshold, int exclude_zero, int* ok, char* issues,
                    int cap);
/* apply_layer_aware_finetuning (predictor.cpp:188-199) on a noisy profile's
   per-layer accuracies (raised in place to the threshold h) -> fine_tuned[n]. */
int moe_apply_finetuning(double* per_layer_accuracy, int n, double threshold, int32_t* fine_tuned);
/* coefficient_of_variation / serverful_cost (cost_model.cpp:124-139); -1 on error. */
double moe_coefficient_of_variation(const double* values, int n);
double moe_serverful_cost(double total_ms, int num_layers, int num_experts, double expert_mem_mb, double m_misc_mb);

/* route_tokens (workload.hpp:90-92) and the popularity profile behind it */
int moe_route_tokens(int64_t tokens, int layer, long iteration, int num_experts, int num_layers,
                     double zipf_s, uint64_t seed, int top_k, int drift_period,
                     int64_t* loads_out);
int moe_popularity(int num_experts, int num_layers, double zipf_s, uint64_t seed, int layer,
                   long iteration, int drift_period, int32_t* perm_out, double* weights_out);

/* --------------------------------------------------- synthetic inputs (host) */
/* Deterministic Zipf-skewed gate inputs on an exactly representable grid
   (DESIGN.md §Synthetic inputs), so ids/counts are bit-exact CPU vs GPU. */
uint64_t moe_stream_key(uint64_t seed, uint64_t a, uint64_t b, uint64_t tag);
int moe_synth_tokens(uint64_t key, int64_t first_token, int64_t tokens, int d_model,
                     int num_experts, uint16_t* x_out);
int moe_synth_gate(uint64_t key, int d_model, int num_experts, const double* popularity,
                   const int32_t* noise_perm, uint16_t* wg_out);
int moe_synth_expert(uint64_t key, int d_model, int d_ff, uint16_t* w1, uint16_t* w3,
                     uint16_t* w2);

#ifdef __cplusplus
}
#endif
#endif /* MOE_B200_H_ */
