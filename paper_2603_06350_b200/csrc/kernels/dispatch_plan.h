// dispatch_plan.h — the per-layer exchange/dispatch plan shared by the host
// planner (exchange_plan.cpp) and the device kernels (dispatch.cu,
// ffn_gemm.cu).  Plain-old-data so it is uploaded with one async H2D copy.
#pragma once
#include <cstdint>

namespace moe {

constexpr int kMaxExperts = 256;
constexpr int kMaxReplicas = 512;
// Row code = (target << 28) | row.  The target indexes a table of row
// buffers (RowTargets): 0 = this rank's received rows / expert outputs,
// 8 = the send / return buffer of the NCCL exchange (kRemoteBit), and in the
// peer-memory exchange g = rank g's buffers, written / read over NVLink.
constexpr int kTargetShift = 28;
constexpr uint32_t kRowMask = (1u << kTargetShift) - 1u;
constexpr uint32_t kRemoteBit = 0x80000000u;  // target 8: the NCCL send/return buffer
constexpr int kSendTarget = 8;
constexpr int kMaxTargets = 16;

struct RowTargets {
  void* base[kMaxTargets];
};

// Peer-memory exchange: after its last row store, the dispatch grid publishes
// `epoch` in flags[g][kind * 8 + src] of every rank g (G == 0: no signal).
struct PeerSignal {
  uint32_t* flags[8];
  uint32_t* counter;      // CTAs finished (self-resetting)
  const uint32_t* epoch;  // the forward's epoch (device memory)
  int G, src, kind, pad;
};

// A layer's placement as the device planner reads it (ScalingPlan.replica_counts
// flattened to rep_base, Placement.gpu_for to gpu_of; types.hpp:59,
// placer.hpp:17).  Uploaded when the host planner decides it — for
// MOE_PLAN_PREDICTED d layers before the layer runs.
struct PlacementTable {
  int E, R, pad0, pad1;
  int rep_base[kMaxExperts + 4];
  int gpu_of[kMaxReplicas];
  int expert_of[kMaxReplicas];
  int slot_of[kMaxExperts];  // this rank's weight slot of expert e (MOE_RESIDENCY_PLACED; else e)
};

// One GEMM segment = the rows of one replica placed on this rank.
struct GemmSeg {
  int row_start;  // first row in the received (permuted) buffer
  int rows;       // > 0
  int slot;       // expert whose weights the replica runs
  int pad;
};

// Single GPU: the combine fused into GEMM2's epilogue.  Every expert-output
// row knows its (token, slot) (row_owner, written by the dispatch kernel); the
// last of a token's k rows to finish an n tile sums the k rows of that tile in
// slot order — the combine kernel's arithmetic — and writes y.
struct FusedCombine {
  const int32_t* row_owner;  // [rows] t * k + j; nullptr: no fusion (separate combine kernel)
  const uint32_t* row_code;  // [T * k] (token, slot) -> row
  const float* wts;          // [T * k]
  int32_t* counters;         // [T * n_tiles] arrivals per (token, n tile); zero between forwards
  void* y;                   // [T, d] bf16
  int k, pad;
};

struct DevPlan {
  int E, R, G, rank;
  int nseg;        // GEMM segments on this rank (replicas here with rows > 0)
  int rows_local;  // rows this rank computes (sum of its segments)
  int rows_send;   // rows this rank ships to other ranks
  int pad0;
  int n_e[kMaxExperts];               // assignments of expert e over all ranks
  int src_off[kMaxExperts];           // this rank's first global rank in expert e
  int rep_base[kMaxExperts + 4];      // flat replica id of (e, 0); [E] = R
  int rep_row_base[kMaxReplicas];     // row(gr) = rep_row_base[f] + gr
  int rep_remote[kMaxReplicas];       // row-code target of replica f's rows (0 local)
  GemmSeg segs[kMaxReplicas];
};

}  // namespace moe
