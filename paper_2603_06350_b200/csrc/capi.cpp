// capi.cpp — the MoE layer forward behind the C-ABI (include/moe_b200.h):
// per layer, on the context's stream (enqueue_forward)
//
//   K1 gate + top-k + histogram (+K2 predictor)        gate.cu
//   G > 1: counts exchange (peer slabs, or NCCL all-gather)
//   plan: on the device (G = 1, or placement planned ahead) or on the host
//         (scale_experts / place_experts on the actual loads, exchange plan)
//   block prefix + K3 dispatch (peer stores at G > 1)  dispatch.cu
//   K4 GEMM1 (SwiGLU) + GEMM2                          ffn_gemm.cu  (tcgen05/TMEM/TMA)
//   K5 combine (peer loads at G > 1)                   dispatch.cu
//
// plus the staged forward (external transport) and the host-buffer calls.
// Replaces layer_forward_time (proj/src/cost_model.cpp:91-122) for callers
// that want the real layer instead of the analytic model.  Context, weights
// and placement: capi_ctx.cpp.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "ctx_internal.h"

namespace moe {
thread_local std::string g_last_error;

// mirror: the gate's last CTA also copies the histograms (gate + predictor,
// `stride` ints) into mapped host memory for the host planner (single GPU)
// Returns true when the histograms still have to be mirrored to the host (the
// tcgen05 gate leaves that to a side-stream copy, off the layer's critical path).
bool stage_gate(moe_ctx* c, Layer& L, const uint16_t* x, int T, cudaStream_t s, int32_t* pred_counts,
                bool mirror = false, int stride = 0) {
  CU_CHECK(cudaMemsetAsync(c->counts.p, 0, sizeof(int32_t) * c->count_stride, s));
  if (c->ext_route) {  // caller-given routing (moe_layer_forward_ids) instead of K1
    CU_CHECK(launch_route_ids(c->ext_ids, c->ext_wts, T, c->E, c->k, c->ids.p, c->wts.p, c->counts.p,
                              c->block_counts.p, c->ids_err, s));
    return false;
  }
  require(L.has_gate, "gate weights not set for layer");
  if (c->fp32) {
    CU_CHECK(launch_gate_f32(reinterpret_cast<const float*>(x), T, c->d, reinterpret_cast<const float*>(L.wg.p), c->E,
                             c->k, c->ids.p, c->wts.p, c->counts.p, c->block_counts.p, s));
    return false;
  }
  // prefill: the tcgen05 gate (128-token tiles of x through TMA); one x map per (x, T)
  const int n_pred_used = pred_counts ? c->n_pred : 0;
  const int Etot = c->E * (1 + n_pred_used);
  const bool mlp = L.pred_w2.p != nullptr && (L.mlp_mask & ((n_pred_used >= 32 ? 0u : (1u << n_pred_used)) - 1u)) != 0;
  if (gate_tc_applies(T, c->d, Etot, c->k, mlp)) {
    if (c->tmGateTc_ptr != x || c->tmGateTc_T != T) {
      c->tmGateTc = make_kmajor_map(x, T, c->d, 128);
      c->tmGateTc_ptr = x;
      c->tmGateTc_T = T;
    }
    const CUtensorMap tmw = make_kmajor_map(L.wg.p, Etot, c->d, Etot <= 16 ? 16 : 32);  // rows past Etot: zero fill
    CU_CHECK(launch_gate_tc(&c->tmGateTc, &tmw, T, c->d, c->E, n_pred_used, c->k, c->ids.p, c->wts.p, c->counts.p,
                            c->block_counts.p, pred_counts ? pred_counts : c->pred_counts.p, nullptr, stride,
                            c->gate_ticket.p, c->num_sms, s, c->front_trace.p));
    return mirror;
  }
  // the prefill gate streams x through TMA boxes: one map per (x, T), rebuilt when they change
  const CUtensorMap* tmx = nullptr;
  if (T >= 148 * 32 && c->d % 512 == 0) {
    if (c->tmGate_ptr != x || c->tmGate_T != T) {
      c->tmGate = make_kmajor_map(x, T, c->d, 32);
      c->tmGate_ptr = x;
      c->tmGate_T = T;
    }
    tmx = &c->tmGate;
  }
  CU_CHECK(launch_gate_topk(reinterpret_cast<const __nv_bfloat16*>(x), T, c->d,
                            reinterpret_cast<const __nv_bfloat16*>(L.wg.p), c->E, pred_counts ? c->n_pred : 0,
                            c->k, c->ids.p, c->wts.p, c->counts.p, c->block_counts.p,
                            pred_counts ? pred_counts : c->pred_counts.p, c->gate_partial.p, s,
                            mirror ? c->h_counts : nullptr, stride, c->gate_ticket.p, L.pred_w2.p, L.mlp_mask, tmx));
  return false;
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
  } else if (plan_mode == MOE_PLAN_PREDICTED && L.plan_for != iteration && L.boot_ready) {
    // the bootstrap placement planned at the previous forward's flush (below)
    L.boot_ready = false;
    L.plan_source = 3;
    ++L.bootstraps;
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
  // MoEless plans off the critical path.  A layer no predictor reaches (l < d)
  // bootstraps from its load history (simulator.cpp:146-151) — and the history
  // is all that needs, so the placement of its NEXT forward is planned here, and
  // that forward takes the device-planned path instead of a host round trip.
  // The target total is this batch's (the reference takes the incoming batch's:
  // the same for fixed batch sizes).  Not with PLACED residency: the copies a
  // new placement may start must be ordered after this forward's GEMMs.
  const bool upstream = layer >= c->pred_distance && c->n_pred > 0 &&
                        c->layers[layer - c->pred_distance].has_pred_weights;
  L.boot_ready = false;
  if (plan_mode == MOE_PLAN_PREDICTED && !upstream && !c->placed) {
    moeless::PredictorProfile hp;
    hp.kind = moeless::PredictorKind::historical;
    const auto guess = moeless::predict({layer, total}, L.history, hp, iteration + 1, 1);
    plan_layer(c, layer, guess.loads, iteration + 1);
    L.boot_ready = true;
  }
}

// local_plan (single GPU): the scan launch also builds the dispatch plan from
// the gate histogram on the device (one extra CTA)
void stage_dispatch(moe_ctx* c, const uint16_t* x, int T, cudaStream_t s, bool upload_plan = true,
                    bool gather = false, bool fused = false, bool local_plan = false) {
  if (upload_plan)
    CU_CHECK(launch_small_copy(c->dplan.p, c->hplan, sizeof(DevPlan), s));  // SM copy from mapped pinned memory
  const int nblk = gate_num_blocks(T);
  // single GPU, few blocks (decode): the dispatch grid builds prefix + plan itself
  const bool fuse_plan = local_plan && !gather && !fused && c->fuse_plan && dispatch_fuses_plan(T);
  if (!fuse_plan)
    CU_CHECK(launch_block_prefix(c->block_counts.p, nblk, c->E, c->dplan.p, c->block_pre.p, s,
                                 local_plan ? c->counts.p : nullptr, c->pdl_prefix()));
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
                           fused ? c->row_owner.p : nullptr, c->pdl_prefix(), fuse_plan ? c->counts.p : nullptr,
                           c->block_counts.p, c->dplan.p));
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
  if (!c->transport) return;  // MOE_EXCHANGE_EXTERNAL: the caller moves the chunks
  // one message per (peer, replica) chunk, in the plan's order on both sides:
  // forward  = my send buffer -> the owners' received-rows buffers,
  // backward = my expert outputs -> the sources' return buffers
  const size_t w = static_cast<size_t>(c->xw);  // row width in 16-bit units (bf16 or fp32 rows)
  const size_t row_bytes = w * 2;
  std::vector<Msg> sends, recvs;
  const auto& out = forward ? c->plan.sends : c->plan.recvs;
  const auto& in = forward ? c->plan.recvs : c->plan.sends;
  uint16_t* out_base = forward ? c->send.p : c->yp.p;
  uint16_t* in_base = forward ? c->xp.p : c->ret.p;
  for (const Chunk& ch : out) sends.push_back(Msg{out_base + ch.row_offset * w, ch.rows * row_bytes, ch.peer});
  for (const Chunk& ch : in) recvs.push_back(Msg{in_base + ch.row_offset * w, ch.rows * row_bytes, ch.peer});
  c->transport->exchange(sends, recvs, s);
}

// K4: which = 0 -> GEMM1 (X -> H, SwiGLU epilogue), 1 -> GEMM2 (H -> Y).
// Prefill default: the 2-SM (cta_group::2, 256-row tile) kernel, launched
// programmatically like the 1-SM kernel (it lost ~4% to it under the 1 kW cap
// before it had PDL, profiles/ab_gemm_variants_r01.md; with PDL it wins,
// profiles/ab_2sm_pdl_r02.md).  MOE_GEMM_VARIANT=1sm / mc select the 1-SM
// kernel or its cluster-multicast form.
// Swap-AB tiles (weights as the M operand, tokens as N; GEMM1 and GEMM2 in one
// launch): 64-token tiles when the batch leaves a few dozen rows per expert
// (decode: 128-row tiles would be mostly padding), 128-token tiles for
// mid-size batches (same MMA work per stage as the 1-SM kernel, no tail
// between the GEMMs).  Returns the tile's token rows, 0 = the 128/256-row kernels
// (profiles/ab_swap_r01.md).
int use_swap(const moe_ctx* c, int T) {
  if (c->fp32 || T <= 0 || c->gemm_variant == 1 || c->gemm_variant == 2 || c->gemm_variant == 3 ||
      c->gemm_variant == 7)
    return 0;
  const int64_t mean_rows = static_cast<int64_t>(T) * c->k * c->G / std::max(1, c->E);  // balanced EP
  if (c->gemm_variant == 5) return 64;
  if (c->gemm_variant == 6) return 128;
  if (c->gemm_variant == 4) return mean_rows <= 64 ? 64 : 128;
  if (mean_rows <= c->swap_rows) return 64;
  return mean_rows <= c->swap128_rows ? 128 : 0;
}

void launch_ffn_gemm(moe_ctx* c, int layer, int which, cudaStream_t s, int64_t rows = 0, bool gather = false,
                     uint16_t* fused_y = nullptr, uint16_t* y2 = nullptr) {
  Layer& L = c->layers[layer];
  const int sn = gather || fused_y ? 0 : use_swap(c, c->gemm_T);
  if (sn) {
    // fused: the GEMM1 call launches both GEMMs, the GEMM2 call adds nothing
    if (c->swap_fuse && which == 1) return;
    CU_CHECK(launch_grouped_gemm_swap(c->swap_fuse ? 2 : which, sn, &c->tmA1s, &L.tmB1, &c->tmA2s, &L.tmB2,
                                      c->dplan.p->segs, &c->dplan.p->nseg, c->d, c->ff, 2 * c->ff, c->d,
                                      reinterpret_cast<__nv_bfloat16*>(c->h.p),
                                      reinterpret_cast<__nv_bfloat16*>(c->yp.p), c->swap_ready.p,
                                      static_cast<int>(c->swap_ready.n), c->num_sms, s, c->use_pdl,
                                      c->swap_half2 ? &L.tmB2h : nullptr));
    return;
  }
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
  if (c->gemm_variant == 7) {  // cluster pairs sharing B through TMA multicast
    const int n = which == 0 ? 2 * c->ff : c->d, kk = which == 0 ? c->d : c->ff;
    CU_CHECK(launch_grouped_gemm_mc(which == 0 ? 0 : 1, which == 0 ? &c->tmA1 : &c->tmA2,
                                    which == 0 ? &L.tmB1h : &L.tmB2h, c->dplan.p->segs, &c->dplan.p->nseg, n, kk, n,
                                    reinterpret_cast<__nv_bfloat16*>(which == 0 ? c->h.p : c->yp.p),
                                    which == 0 ? c->ff : c->d, c->num_sms, s, c->use_pdl, c->group_m[which]));
    return;
  }
  // default (auto) for batches past the swap-AB range: the 2-SM cta_group::2
  // kernel (256-row tiles, B split across the SM pair, PDL behind its
  // producer) — +4-5% tokens/s at cfg2 over the 1-SM kernel in short and
  // 150-step runs alike (profiles/ab_2sm_pdl_r02.md); the 1-SM kernel keeps the
  // opt-in gather / fused-combine / dynamic-scheduler paths
  const bool two_sm = c->gemm_variant == 2 || (c->gemm_variant == 0 && !gather && !fused_y);
  const bool m256 = c->gemm_variant == 3;
  if (two_sm) {
    if (which == 0)
      CU_CHECK(launch_grouped_gemm_2sm(0, &c->tmA1, &L.tmB1h, c->dplan.p->segs, &c->dplan.p->nseg, 2 * c->ff, c->d,
                                       2 * c->ff, reinterpret_cast<__nv_bfloat16*>(c->h.p), c->ff, c->num_sms, s,
                                       c->use_pdl, c->group_m[0], c->sched_2sm() ? c->gemm_sched.p : nullptr));
    else
      CU_CHECK(launch_grouped_gemm_2sm(1, &c->tmA2, &L.tmB2h, c->dplan.p->segs, &c->dplan.p->nseg, c->d, c->ff, c->d,
                                       reinterpret_cast<__nv_bfloat16*>(c->yp.p), c->d, c->num_sms, s, c->use_pdl,
                                       c->group_m[1], c->sched_2sm() ? c->gemm_sched.p + 2 : nullptr,
                                       c->row_owner.p, c->wts.p, reinterpret_cast<__nv_bfloat16*>(y2), c->comb_cnt.p));
    return;
  }
  if (m256) {
    auto fn = launch_grouped_gemm_m256;
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
  int* sched = c->sched_1sm() ? c->gemm_sched.p + 2 * which : nullptr;
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
                          c->num_sms, s, c->pdl_combine()));
}

// invalid caller ids (moe_layer_forward_ids), flagged by route_ids_kernel
void check_ids(moe_ctx* c) {
  if (!c->ids_err || *reinterpret_cast<volatile int*>(c->ids_err) == 0) return;
  const int t = *c->ids_err - 1;
  *c->ids_err = 0;
  throw std::invalid_argument("routing ids of token " + std::to_string(t) +
                              " are invalid (expert out of range or chosen twice)");
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
  check_ids(c);
  stage_plan(c, c->pending.layer, c->pending.mode, c->pending.iteration, c->h_counts, c->pending.stride);
  if (c->pending.gemm_slot >= 0) c->gemm_rows[c->pending.gemm_slot] = c->plan.rows_local;
}

// GEMM2 writes y itself (combine fused, FusedY in ffn_gemm.cu): top-2 on one
// GPU on the 2-SM prefill kernel — the same conditions launch_ffn_gemm uses to
// pick that kernel, decided once per forward for dispatch, GEMM2 and combine.
bool fused_y_2sm(moe_ctx* c, int T, bool gather, bool fused) {
  return c->fuse_y && c->G == 1 && !c->p2p && !c->fp32 && c->k == 2 && T > 0 && !gather && !fused &&
         !c->ext_route && (c->gemm_variant == 0 || c->gemm_variant == 2) && use_swap(c, T) == 0 &&
         static_cast<int64_t>(T) <= c->Tmax;
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
  c->gemm_T = T;
  const bool swap = use_swap(c, T) != 0;
  const bool gather = c->gather && c->G == 1 && !c->fp32 && (c->gemm_variant == 0 || c->gemm_variant == 1) && T > 0 &&
                      !swap;
  // single GPU, bf16, 1-SM K4: the combine runs inside GEMM2's epilogue
  const bool fused =
      c->fuse_combine && c->G == 1 && !c->fp32 && (c->gemm_variant == 0 || c->gemm_variant == 1) && !swap;
  if (gather && (c->tmX_ptr != x || c->tmX_T != T)) {
    c->tmX = make_kmajor_map(x, T, c->d, 1);
    c->tmX_ptr = x;
    c->tmX_T = T;
  }
  mark(0);
  if (c->trace_marker) CU_CHECK(launch_trace_marker(s));
  // decode: pull the first experts' weights into L2 on a side stream while the
  // front end runs (the swap-AB K4 streams them in expert order)
  const bool prefetch = swap && c->prefetch_mb > 0 && c->G == 1 && !c->fp32 && L.w13.p;
  const size_t prefetch_bytes =
      prefetch ? std::min(static_cast<size_t>(c->prefetch_mb) << 20, L.w13.n * sizeof(uint16_t)) : 0;
  // single GPU, small batch: gate, top-k, plan and dispatch in one cooperative
  // launch (kernels/frontend.cu)
  const int Etot = with_pred ? c->count_stride : c->E;
  const bool front = c->frontend && c->G == 1 && !c->fp32 && !c->ext_route && !gather && !fused && L.has_gate &&
                     frontend_applies(T, c->d, Etot, c->k, c->num_sms);
  const bool inline_prefetch = prefetch && front && c->front_prefetch_inline;
  // (the fused front end does not write the row owners the fused GEMM2 epilogue reads)
  const bool fy = !front && fused_y_2sm(c, T, gather, fused);
  if (prefetch && !inline_prefetch) {
    CU_CHECK(cudaEventRecord(c->ev_pf_fork, s));
    CU_CHECK(cudaStreamWaitEvent(c->pstream, c->ev_pf_fork, 0));
    CU_CHECK(launch_l2_prefetch(L.w13.p, prefetch_bytes, c->pstream));
    CU_CHECK(cudaEventRecord(c->ev_pf_join, c->pstream));
  }
  // the gate publishes the histograms itself (not the caller-ids kernel)
  const bool mirrored = c->G == 1 && !c->fp32 && T > 0 && !c->ext_route;
  bool side_mirror = false;
  if (front) {
    CU_CHECK(launch_frontend(reinterpret_cast<const __nv_bfloat16*>(x), T, c->d,
                             reinterpret_cast<const __nv_bfloat16*>(L.wg.p), c->E, with_pred ? c->n_pred : 0, c->k,
                             c->ids.p, c->wts.p, c->counts.p, c->block_counts.p, c->gate_partial.p, c->h_counts,
                             L.pred_w2.p, L.mlp_mask, reinterpret_cast<__nv_bfloat16*>(c->xp.p), c->row_code.p,
                             c->dplan.p, inline_prefetch ? L.w13.p : nullptr, prefetch_bytes, c->front_trace.p, s));
    // "counts are in host memory" on a side branch: an event node between the
    // front end and the GEMM would cut their programmatic edge
    CU_CHECK(cudaEventRecord(c->ev_front, s));
    CU_CHECK(cudaStreamWaitEvent(c->pstream, c->ev_front, 0));
    CU_CHECK(cudaEventRecordWithFlags(c->ev_counts, c->pstream, rec));
    CU_CHECK(cudaEventRecord(c->ev_pf_join, c->pstream));
    mark(1);
    mark(2);
  } else {
    side_mirror = stage_gate(c, L, x, T, s, with_pred ? c->counts.p + c->E : nullptr, mirrored, stride);
    if (side_mirror) {
      // the histograms to mapped host memory on the side stream: the PCIe writes
      // and their flush stay off the layer's critical path
      CU_CHECK(cudaEventRecord(c->ev_front, s));
      CU_CHECK(cudaStreamWaitEvent(c->pstream, c->ev_front, 0));
      CU_CHECK(launch_small_copy(c->h_counts, c->counts.p, pad16(sizeof(int32_t) * stride), c->pstream));
      CU_CHECK(cudaEventRecordWithFlags(c->ev_counts, c->pstream, rec));
      CU_CHECK(cudaEventRecord(c->ev_pf_join, c->pstream));
    }
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
      require(c->transport != nullptr, "staged API required for external exchange");
      c->transport->all_gather(c->counts.p, c->counts_all.p, stride, s);
      CU_CHECK(launch_small_copy(c->h_counts, c->counts_all.p, pad16(sizeof(int32_t) * c->G * stride), s));
    } else if (!mirrored) {
      CU_CHECK(launch_small_copy(c->h_counts, c->counts.p, pad16(sizeof(int32_t) * stride), s));
    }
    if (deferred) {
      if (!side_mirror) CU_CHECK(cudaEventRecordWithFlags(c->ev_counts, s, rec));
      mark(1);
      if (c->G > 1) CU_CHECK(launch_plan_exchange(c->counts_all.p, stride, c->G, c->rank, L.ptab.p, c->dplan.p, s));
      mark(2);
      stage_dispatch(c, x, T, s, /*upload_plan=*/false, gather, fused || fy, /*local_plan=*/c->G == 1);
    } else {
      mark(1);
      CU_CHECK(cudaStreamSynchronize(s));  // the host plans on the real histogram
      check_p2p(c);
      check_ids(c);
      stage_plan(c, layer, plan_mode, iteration, c->h_counts, stride);
      mark(2);
      stage_dispatch(c, x, T, s);  // uploads the plan; P2P rows land in their owners' buffers
    }
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
  launch_ffn_gemm(c, layer, 1, s, rows, false, fused ? y : nullptr, fy ? y : nullptr);
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
  if (!fused && !fy && !c->skip_combine) stage_combine(c, y, T, s);
  if (prefetch || front || side_mirror) CU_CHECK(cudaStreamWaitEvent(s, c->ev_pf_join, 0));  // the side stream rejoins
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
  // A caller stream: context uploads (placement table, staged gate weights,
  // weights) are enqueued on c->stream, so the forward first waits for them,
  // and later uploads wait for the forward (ForeignStreamOrder's destructor)
  struct ForeignStreamOrder {
    moe_ctx* c;
    cudaStream_t s;
    ~ForeignStreamOrder() {
      if (s != c->stream && cudaEventRecord(c->ev_fwd_tail, s) == cudaSuccess)
        cudaStreamWaitEvent(c->stream, c->ev_fwd_tail, 0);
    }
  } order{c, s};
  if (s != c->stream) {
    CU_CHECK(cudaEventRecord(c->ev_ctx_tail, c->stream));
    CU_CHECK(cudaStreamWaitEvent(s, c->ev_ctx_tail, 0));
  }
  // the fused predictor (K2) runs when the layer has predictor weights: its
  // histograms follow the gate's in the same counts buffer
  const bool with_pred = c->n_pred > 0 && L.has_pred_weights && !c->ext_route;
  const int stride = with_pred ? c->count_stride : c->E;
  const bool ahead = c->G > 1 && c->p2p && !c->fp32 &&
                     (plan_mode == MOE_PLAN_FIXED ||
                      (plan_mode == MOE_PLAN_PREDICTED && (L.plan_for == iteration || L.boot_ready)));
  if (ahead) ensure_placement(c, layer);
  if (c->user_capture) {
    // recorded into the caller's multi-forward graph (moe_graph_begin)
    require(s == c->stream, "moe_graph_begin: forwards inside a capture must use the context's stream");
    require(!timed, "moe_graph_begin: stats cannot be taken inside a capture");
    require((c->G == 1 || ahead) && !c->placed && !c->ext_route,
            "moe_graph_begin: only device-planned forwards (G == 1, or FIXED / PREDICTED ahead) can be captured");
    enqueue_forward(c, L, layer, x, T, y, plan_mode, iteration, s, with_pred, stride, x_consumed, ahead, true,
                    [](int) {});
    return;
  }
  if (c->use_graphs && !timed && (c->G == 1 || ahead) && !c->placed && !c->ext_route) {
    // Replay the layer's whole device sequence (8-14 kernels) as one CUDA
    // graph: captured once per (layer, tokens, buffers), then launched with a
    // single call — the launch-bound decode regime pays one launch, not ten.
    const GraphKey key{layer, T, x, y, x_consumed, with_pred, L.mlp_mask};
    auto it = c->graphs.find(key);
    if (it == c->graphs.end()) {
      CU_CHECK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
      c->capturing = true;
      try {
        enqueue_forward(c, L, layer, x, T, y, plan_mode, iteration, s, with_pred, stride, x_consumed, ahead, true,
                        [](int) {});
      } catch (...) {
        c->capturing = false;
        cudaGraph_t dead = nullptr;
        cudaStreamEndCapture(s, &dead);
        if (dead) cudaGraphDestroy(dead);
        throw;
      }
      c->capturing = false;
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
    check_ids(c);
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

}  // namespace moe

extern "C" {

const char* moe_last_error(void) { return g_last_error.c_str(); }

const char* moe_version(void) { return "moe_b200 0.1.0 (sm_100a)"; }

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
                              c->gate_partial.p, s, nullptr, 0, nullptr, L.pred_w2.p, L.mlp_mask));
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
                              c->wts.p, c->counts.p, c->block_counts.p, pred_counts, c->gate_partial.p, s, nullptr,
                              0, nullptr, L.pred_w2.p, L.mlp_mask));
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

int moe_graph_begin(moe_ctx* c) {
  return guarded([&] {
    require(c != nullptr, "null argument");
    require(!c->user_capture, "moe_graph_begin: a capture is already open");
    CU_CHECK(cudaSetDevice(c->desc.device));
    flush_pending_plan(c);  // the previous forward's planner work, before the stream is captured
    CU_CHECK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    c->user_capture = true;
    c->capturing = true;
  });
}

int moe_graph_end(moe_ctx* c, int* graph_id) {
  return guarded([&] {
    require(c && graph_id, "null argument");
    require(c->user_capture, "moe_graph_end: no capture is open");
    c->user_capture = false;
    c->capturing = false;
    cudaGraph_t g = nullptr;
    const cudaError_t e = cudaStreamEndCapture(c->stream, &g);
    if (e != cudaSuccess) {
      if (g) cudaGraphDestroy(g);
      CU_CHECK(e);
    }
    cudaGraphExec_t ex = nullptr;
    const cudaError_t ei = cudaGraphInstantiate(&ex, g, 0);
    cudaGraphDestroy(g);
    CU_CHECK(ei);
    CU_CHECK(cudaGraphUpload(ex, c->stream));
    c->user_graphs.push_back(ex);
    *graph_id = static_cast<int>(c->user_graphs.size()) - 1;
  });
}

int moe_graph_launch(moe_ctx* c, int graph_id, void* stream) {
  return guarded([&] {
    require(c != nullptr, "null argument");
    require(graph_id >= 0 && graph_id < static_cast<int>(c->user_graphs.size()), "moe_graph_launch: unknown graph");
    require(!c->user_capture, "moe_graph_launch: a capture is open");
    CU_CHECK(cudaSetDevice(c->desc.device));
    cudaStream_t s = pick(c, stream);
    if (s != c->stream) {  // after the context's uploads; later uploads after the replay
      CU_CHECK(cudaEventRecord(c->ev_ctx_tail, c->stream));
      CU_CHECK(cudaStreamWaitEvent(s, c->ev_ctx_tail, 0));
    }
    CU_CHECK(cudaGraphLaunch(c->user_graphs[graph_id], s));
    if (s != c->stream) {
      CU_CHECK(cudaEventRecord(c->ev_fwd_tail, s));
      CU_CHECK(cudaStreamWaitEvent(c->stream, c->ev_fwd_tail, 0));
    }
  });
}

int moe_layer_forward_ids(moe_ctx* c, int layer, const uint16_t* x, const int32_t* ids, const float* weights,
                          int T, uint16_t* y, int plan_mode, long iteration, moe_layer_stats* stats, void* stream) {
  return guarded([&] {
    require(c && (T == 0 || (x && y && ids)), "null argument");
    require(c->k <= c->E, "top_k exceeds num_experts");
    struct Restore {
      moe_ctx* c;
      ~Restore() { c->ext_route = false, c->ext_ids = nullptr, c->ext_wts = nullptr; }
    } restore{c};
    c->ext_route = true;
    c->ext_ids = ids;
    c->ext_wts = weights;
    forward_device(c, layer, x, T, y, plan_mode, iteration, stats, pick(c, stream));
  });
}

int moe_last_plan(moe_ctx* c, int32_t* n_e, int32_t* segs, int max_segs, int* nseg, int64_t* rows_local) {
  return guarded([&] {
    require(c && nseg, "null argument");
    CU_CHECK(cudaSetDevice(c->desc.device));
    CU_CHECK(cudaStreamSynchronize(c->stream));
    flush_pending_plan(c);
    DevPlan p;
    CU_CHECK(cudaMemcpy(&p, c->dplan.p, sizeof(DevPlan), cudaMemcpyDeviceToHost));
    require(p.nseg <= max_segs || !segs, "segment array too small");
    if (n_e)
      for (int e = 0; e < c->E; ++e) n_e[e] = p.n_e[e];
    if (segs)
      for (int i = 0; i < p.nseg; ++i) {
        segs[3 * i] = p.segs[i].row_start;
        segs[3 * i + 1] = p.segs[i].rows;
        segs[3 * i + 2] = p.segs[i].slot;
      }
    *nseg = p.nseg;
    if (rows_local) *rows_local = p.rows_local;
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
    c->gemm_T = T;
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
      case 12: *ptr = c->front_trace.p; r = c->front_trace.p ? 148 : 0; break;  // MOE_FRONT_TRACE stamps [148][16] u64
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

}  // extern "C"
