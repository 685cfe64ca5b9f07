// capi_ctx.cpp — context lifetime, peer-memory slab exchange, weights, gates,
// placement and expert weight residency behind the C-ABI (include/moe_b200.h).
#include <cuda.h>
#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "ctx_internal.h"

namespace moe {

NcclApi g_nccl;

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
  // transactional: if the placement cannot be made resident (PLACED), the
  // layer keeps its previous placement and the registry does not record it
  std::vector<int32_t> old_counts = L.rep_counts, old_gpu = L.rep_gpu;
  const bool had = L.has_placement;
  L.rep_counts.assign(sp.replica_counts.begin(), sp.replica_counts.end());
  L.rep_gpu.clear();
  for (auto& v : pr.placement.gpu_for) L.rep_gpu.insert(L.rep_gpu.end(), v.begin(), v.end());
  try {
    placement_changed(c, layer);
  } catch (...) {
    L.rep_counts.swap(old_counts);
    L.rep_gpu.swap(old_gpu);
    L.has_placement = had;
    throw;
  }
  moeless::update_registry(c->registry, pr.placement, iteration);
  L.warm = pr.warm_count;
  L.cold = pr.cold_count;
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

}  // namespace moe

extern "C" {

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
    if (const char* v = std::getenv("MOE_GEMM_SCHED")) c->sched_mode = std::string(v) == "dynamic" ? 2 : std::string(v) == "static" ? 1 : 0;
    if (const char* v = std::getenv("MOE_PDL")) c->use_pdl = std::string(v) != "0";
    if (const char* v = std::getenv("MOE_GATHER")) c->gather = std::string(v) == "1";
    if (const char* v = std::getenv("MOE_FUSED_COMBINE")) c->fuse_combine = std::string(v) == "1";
    if (const char* v = std::getenv("MOE_FUSED_Y")) c->fuse_y = std::string(v) != "0";
    if (const char* v = std::getenv("MOE_GEMM_GROUP_M")) std::sscanf(v, "%d,%d", &c->group_m[0], &c->group_m[1]);
    if (const char* v = std::getenv("MOE_GEMM_VARIANT")) {
      const std::string s(v);
      c->gemm_variant = s == "1sm"      ? 1
                        : s == "2sm"    ? 2
                        : s == "m256"   ? 3
                        : s == "swap"   ? 4
                        : s == "swap64" ? 5
                        : s == "swap128" ? 6
                        : s == "mc"     ? 7
                                         : 0;
    }
    if (const char* v = std::getenv("MOE_GEMM_SWAP_ROWS")) c->swap_rows = std::atoi(v);
    if (const char* v = std::getenv("MOE_GEMM_SWAP128_ROWS")) c->swap128_rows = std::atoi(v);
    if (const char* v = std::getenv("MOE_SWAP_FUSE")) c->swap_fuse = std::string(v) != "0";
    if (const char* v = std::getenv("MOE_SWAP_HALF2")) c->swap_half2 = std::string(v) != "0";
    if (const char* v = std::getenv("MOE_FUSE_PLAN")) c->fuse_plan = std::string(v) != "0";
    if (const char* v = std::getenv("MOE_FRONTEND")) c->frontend = std::string(v) != "0";
    if (const char* v = std::getenv("MOE_DEBUG_SKIP_COMBINE")) c->skip_combine = std::string(v) == "1";
    if (const char* v = std::getenv("MOE_FRONT_PREFETCH")) c->front_prefetch_inline = std::string(v) == "inline";
    if (const char* v = std::getenv("MOE_FRONT_TRACE"); v && (std::string(v) == "1" || std::string(v) == "2")) {
      c->trace_marker = std::string(v) == "2";
      c->front_trace.alloc(148 * 16);
      CU_CHECK(cudaMemset(c->front_trace.p, 0, 148 * 16 * sizeof(unsigned long long)));
      CU_CHECK(set_swap_trace(c->front_trace.p));
      CU_CHECK(set_combine_trace(c->front_trace.p));
    }
    if (const char* v = std::getenv("MOE_DECODE_PREFETCH_MB")) c->prefetch_mb = std::max(0, std::atoi(v));
    if (const char* v = std::getenv("MOE_PDL_FRONT")) c->pdl_front = std::atoi(v);
    if (const char* v = std::getenv("MOE_SWAP_WPOL")) g_swap_wpol.store(std::atoi(v));
    if (const char* v = std::getenv("MOE_GEMM_L2POL")) g_gemm_l2pol.store(std::atoi(v));
    if (const char* v = std::getenv("MOE_GATE_MAX_SPLITS")) g_gate_max_splits.store(std::max(1, std::atoi(v)));
    if (const char* v = std::getenv("MOE_GATE_CLUSTER")) g_gate_cluster.store(std::atoi(v) != 0);
    if (const char* v = std::getenv("MOE_GATE_STREAM")) g_gate_stream.store(std::atoi(v) != 0);
    if (const char* v = std::getenv("MOE_GATE_TC")) g_gate_tc.store(std::atoi(v) != 0);
    if (const char* v = std::getenv("MOE_GATE_TC_BKS")) g_gate_tc_bks.store(std::atoi(v));
    if (const char* v = std::getenv("MOE_GATE_MIN_SPLITS")) g_gate_min_splits.store(std::max(1, std::atoi(v)));
    if (const char* v = std::getenv("MOE_P2P_TIMEOUT_MS")) c->p2p_timeout_ns = std::strtoull(v, nullptr, 10) * 1000000ull;
    require(D.exchange_mode >= MOE_EXCHANGE_NCCL && D.exchange_mode <= MOE_EXCHANGE_COPY, "unknown exchange mode");
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
    CU_CHECK(preload_frontend_kernels());
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
    c->gate_ticket.alloc(4);
    CU_CHECK(cudaMemset(c->gate_ticket.p, 0, 4 * sizeof(unsigned)));
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
      c->tmA1s = make_kmajor_map(c->xp.p, c->rows_cap, c->d, 32);
      c->tmA2s = make_kmajor_map(c->h.p, c->rows_cap, c->ff, 32);
      c->swap_ready.alloc(static_cast<size_t>(c->rows_cap) / 64 + kMaxReplicas + 2);
      CU_CHECK(cudaMemset(c->swap_ready.p, 0, c->swap_ready.n * sizeof(int)));
    }
    // mapped pinned control buffers, read/written by small SM copies (UVA pointers)
    CU_CHECK(cudaHostAlloc(&c->hplan, sizeof(DevPlan), cudaHostAllocMapped));
    CU_CHECK(cudaHostAlloc(&c->h_counts, pad16(sizeof(int32_t) * c->count_stride * c->G), cudaHostAllocMapped));
    CU_CHECK(cudaHostAlloc(&c->ids_err, sizeof(int) * 4, cudaHostAllocMapped));
    *c->ids_err = 0;
    c->events.create();
    CU_CHECK(cudaEventCreateWithFlags(&c->ev_counts, cudaEventDisableTiming));
    CU_CHECK(cudaEventCreateWithFlags(&c->ev_ctx_tail, cudaEventDisableTiming));
    CU_CHECK(cudaStreamCreateWithFlags(&c->pstream, cudaStreamNonBlocking));
    CU_CHECK(cudaEventCreateWithFlags(&c->ev_pf_fork, cudaEventDisableTiming));
    CU_CHECK(cudaEventCreateWithFlags(&c->ev_front, cudaEventDisableTiming));
    CU_CHECK(cudaEventCreateWithFlags(&c->ev_pf_join, cudaEventDisableTiming));
    CU_CHECK(cudaEventCreateWithFlags(&c->ev_fwd_tail, cudaEventDisableTiming));
    for (auto& tri : c->gemm_ev)
      for (cudaEvent_t& e : tri) CU_CHECK(cudaEventCreate(&e));
    if (c->G > 1 && D.exchange_mode == MOE_EXCHANGE_NCCL) {
      require(D.nccl_unique_id != nullptr, "nccl_unique_id required for world_size > 1");
      g_nccl.load();
      ncclUniqueId id;
      std::memcpy(&id, D.nccl_unique_id, sizeof(id));
      g_nccl.check(g_nccl.CommInitRank(&c->comm, c->G, id, c->rank), "ncclCommInitRank");
      c->transport = make_nccl_transport(c->comm);
    } else if (c->G > 1 && D.exchange_mode == MOE_EXCHANGE_COPY) {
      c->transport = make_copy_transport(D.nccl_unique_id, c->G, c->rank, D.device, c->p2p_timeout_ns);
    }
    *out = c.release();
  });
}

int moe_ctx_destroy(moe_ctx* c) {
  return guarded([&] {
    if (!c) return;
    cudaSetDevice(c->desc.device);
    cudaStreamSynchronize(c->stream);
    c->transport.reset();
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
    if (c->ids_err) cudaFreeHost(c->ids_err);
    c->events.destroy();
    if (c->hplan) cudaFreeHost(c->hplan);
    if (c->h_counts) cudaFreeHost(c->h_counts);
    if (c->wg_stage) cudaFreeHost(c->wg_stage);
    if (c->ev_wg_staged) cudaEventDestroy(c->ev_wg_staged);
    if (c->ev_counts) cudaEventDestroy(c->ev_counts);
    if (c->ev_ctx_tail) cudaEventDestroy(c->ev_ctx_tail);
    if (c->pstream) {
      cudaStreamSynchronize(c->pstream);
      cudaStreamDestroy(c->pstream);
    }
    for (cudaEvent_t e : {c->ev_pf_fork, c->ev_pf_join, c->ev_front})
      if (e) cudaEventDestroy(e);
    if (c->ev_fwd_tail) cudaEventDestroy(c->ev_fwd_tail);
    for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second);
    for (cudaGraphExec_t g : c->user_graphs) cudaGraphExecDestroy(g);
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

int moe_set_gate_weights_device(moe_ctx* c, int layer, const void* wg_dev, void* stream) {
  return guarded([&] {
    Layer& L = layer_at(c, layer);
    require(wg_dev != nullptr, "null gate weights");
    if (!L.wg.p) {
      L.wg.alloc(static_cast<size_t>(c->E) * c->d * (1 + c->n_pred) * c->elem);
      CU_CHECK(cudaMemsetAsync(L.wg.p, 0, L.wg.n * 2, c->stream));
    }
    // stream-ordered device -> device copy: no staging, no host wait
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : c->stream;
    CU_CHECK(cudaMemcpyAsync(L.wg.p, wg_dev, static_cast<size_t>(c->E) * c->d * 2 * c->elem,
                             cudaMemcpyDeviceToDevice, s));
    L.has_gate = true;
  });
}

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

int moe_set_predictor_mlp(moe_ctx* c, int layer, int slot, const uint16_t* w1, const float* w2) {
  return guarded([&] {
    Layer& L = layer_at(c, layer);
    require(slot >= 0 && slot < c->n_pred, "predictor slot out of range");
    require(slot < 32, "MLP predictor slots are limited to 32");
    if (w1) {
      const int rc = moe_set_predictor_weights(c, layer, slot, w1);
      if (rc != MOE_OK) throw Status{rc, g_last_error};
    }
    CU_CHECK(cudaStreamSynchronize(c->stream));
    if (!w2) {  // back to the linear predictor
      L.mlp_mask &= ~(1u << slot);
      return;
    }
    const size_t EE = static_cast<size_t>(c->E) * c->E;
    if (!L.pred_w2.p) {
      L.pred_w2.alloc(EE * c->n_pred);
      CU_CHECK(cudaMemset(L.pred_w2.p, 0, L.pred_w2.n * sizeof(float)));
    }
    CU_CHECK(cudaMemcpy(L.pred_w2.p + slot * EE, w2, EE * sizeof(float), cudaMemcpyHostToDevice));
    L.mlp_mask |= 1u << slot;
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

int moe_get_placement(moe_ctx* c, int layer, int32_t* rc, int32_t* rg, int max_replicas, int* n_replicas) {
  return guarded([&] {
    Layer& L = layer_at(c, layer);
    require(rc && n_replicas, "null argument");
    flush_pending_plan(c);  // a deferred SYNC plan of the last forward lands first
    ensure_placement(c, layer);
    const int R = static_cast<int>(L.rep_gpu.size());
    require(!rg || R <= max_replicas, "replica array too small");
    for (int e = 0; e < c->E; ++e) rc[e] = L.rep_counts[e];
    if (rg)
      for (int i = 0; i < R; ++i) rg[i] = L.rep_gpu[i];
    *n_replicas = R;
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

}  // extern "C"
