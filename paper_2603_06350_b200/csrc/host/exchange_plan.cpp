// exchange_plan.cpp — integer replica split + the row exchange it implies.
//
// Inputs: every rank's gate histogram counts_all[G][E] (after the counts
// all-gather), the plan's replica counts R_e and the placement's replica ->
// GPU map (ScalingPlan.replica_counts, types.hpp:59; Placement.gpu_for,
// placer.hpp:17).  Output: this rank's DevPlan (uploaded for the dispatch and
// GEMM kernels) and the send/recv chunk lists the NCCL exchange issues.
//
// Rule (making cost_model.cpp:98-106 integer): expert e's
// assignments ordered by (source rank, token) get global ranks 0..n_e-1;
// replica r owns ranks [start_r, start_r + size_r) with size_r = floor(n/R) +
// [r < n mod R].  Because global rank order is source-major, the rows one
// source contributes to one replica are a contiguous sub-range — so every
// (source, replica) pair is ONE contiguous chunk on both sides and the
// receiver places it directly into the replica's segment (no second permute).
// Send order and receive order are both (peer, replica ascending), which is
// what NCCL's in-order p2p matching needs.
#include "exchange_plan.h"

#include <algorithm>
#include <stdexcept>
#include <string>

namespace moe {

void build_exchange_plan(int G, int rank, int E, const int64_t* counts_all, const int32_t* R,
                         const int32_t* gpu_of, HostPlan& out, bool direct) {
  if (G < 1 || rank < 0 || rank >= G) throw std::invalid_argument("bad world size / rank");
  if (E < 1 || E > kMaxExperts) throw std::invalid_argument("num_experts out of range");
  DevPlan& p = out.dev;
  p = DevPlan{};
  p.E = E;
  p.G = G;
  p.rank = rank;
  int f = 0;
  for (int e = 0; e < E; ++e) {
    if (R[e] < 1) throw std::invalid_argument("expert " + std::to_string(e) + " has no replica");
    p.rep_base[e] = f;
    f += R[e];
  }
  if (f > kMaxReplicas) throw std::invalid_argument("too many replicas in one layer");
  p.rep_base[E] = f;
  p.R = f;
  for (int i = 0; i < f; ++i)
    if (gpu_of[i] < 0 || gpu_of[i] >= G)
      throw std::invalid_argument("replica placed on invalid GPU " + std::to_string(gpu_of[i]));

  std::vector<int64_t> n(E, 0), off(static_cast<size_t>(G) * E, 0);
  for (int e = 0; e < E; ++e)
    for (int s = 0; s < G; ++s) {
      off[static_cast<size_t>(s) * E + e] = n[e];
      n[e] += counts_all[static_cast<size_t>(s) * E + e];
    }
  for (int e = 0; e < E; ++e) {
    if (n[e] > INT32_MAX) throw std::invalid_argument("expert load exceeds 2^31");
    p.n_e[e] = static_cast<int>(n[e]);
    p.src_off[e] = static_cast<int>(off[static_cast<size_t>(rank) * E + e]);
  }
  // replica ranges
  out.rep_start.assign(f, 0);
  out.rep_size.assign(f, 0);
  for (int e = 0; e < E; ++e) {
    const int64_t q = n[e] / R[e], rem = n[e] % R[e];
    for (int r = 0; r < R[e]; ++r) {
      const int id = p.rep_base[e] + r;
      out.rep_size[id] = q + (r < rem ? 1 : 0);
      out.rep_start[id] = r * q + std::min<int64_t>(r, rem);
    }
  }
  // segments of this rank (replica order == (expert, ordinal) order)
  out.seg_start.assign(f, -1);
  int64_t rows = 0;
  p.nseg = 0;
  for (int id = 0; id < f; ++id) {
    if (gpu_of[id] != rank) continue;
    out.seg_start[id] = rows;
    p.rep_row_base[id] = static_cast<int>(rows - out.rep_start[id]);
    p.rep_remote[id] = 0;
    if (out.rep_size[id] > 0) {
      int e = 0;
      while (p.rep_base[e + 1] <= id) ++e;
      // Replicas of one expert that sit on the same GPU share its resident
      // weights and occupy adjacent rows: schedule them as ONE grouped-GEMM
      // problem so the weights stream once and only one m-tile is partial.
      GemmSeg* last = p.nseg > 0 ? &p.segs[p.nseg - 1] : nullptr;
      if (last && last->slot == e && last->row_start + last->rows == rows)
        last->rows += static_cast<int>(out.rep_size[id]);
      else
        p.segs[p.nseg++] = GemmSeg{static_cast<int>(rows), static_cast<int>(out.rep_size[id]), e, 0};
    }
    rows += out.rep_size[id];
  }
  out.rows_local = rows;
  out.sends.clear();
  out.recvs.clear();
  int64_t send_rows = 0;
  auto my_range = [&](int s, int e, int id, int64_t& lo, int64_t& hi) {
    const int64_t so = off[static_cast<size_t>(s) * E + e];
    const int64_t sc = counts_all[static_cast<size_t>(s) * E + e];
    lo = std::max(out.rep_start[id], so);
    hi = std::min(out.rep_start[id] + out.rep_size[id], so + sc);
  };
  if (direct) {
    // every GPU lays out its segments the same way (replica order), so each
    // rank can compute where its rows land in any peer's buffer
    std::vector<int64_t> fill(G, 0);
    for (int id = 0; id < f; ++id) {
      const int g = gpu_of[id];
      const int64_t seg = fill[g];
      fill[g] += out.rep_size[id];
      p.rep_remote[id] = g;
      if (g == rank) continue;  // local replicas keep their segment base from above
      if (seg - out.rep_start[id] < INT32_MIN || seg > INT32_MAX)
        throw std::invalid_argument("row count exceeds 2^31");
      p.rep_row_base[id] = static_cast<int>(seg - out.rep_start[id]);
      int e = 0;
      while (p.rep_base[e + 1] <= id) ++e;
      int64_t lo, hi;
      my_range(rank, e, id, lo, hi);
      if (hi > lo) send_rows += hi - lo;
    }
    for (int g = 0; g < G; ++g)
      if (fill[g] > kRowMask) throw std::invalid_argument("row count exceeds the row-code range");
    out.rows_send = send_rows;
    p.rows_local = static_cast<int>(rows);
    p.rows_send = static_cast<int>(send_rows);
    return;
  }
  // sends: my rows bound to replicas elsewhere, peer-major then replica order
  for (int peer = 0; peer < G; ++peer) {
    if (peer == rank) continue;
    for (int e = 0; e < E; ++e)
      for (int id = p.rep_base[e]; id < p.rep_base[e + 1]; ++id) {
        if (gpu_of[id] != peer) continue;
        int64_t lo, hi;
        my_range(rank, e, id, lo, hi);
        p.rep_remote[id] = kSendTarget;
        p.rep_row_base[id] = static_cast<int>(send_rows - lo);
        if (hi > lo) {
          out.sends.push_back({peer, id, send_rows, hi - lo});
          send_rows += hi - lo;
        }
      }
  }
  out.rows_send = send_rows;
  // receives: rows other ranks contribute to my replicas, peer-major, replica order
  for (int peer = 0; peer < G; ++peer) {
    if (peer == rank) continue;
    for (int e = 0; e < E; ++e)
      for (int id = p.rep_base[e]; id < p.rep_base[e + 1]; ++id) {
        if (gpu_of[id] != rank) continue;
        int64_t lo, hi;
        my_range(peer, e, id, lo, hi);
        if (hi > lo) out.recvs.push_back({peer, id, out.seg_start[id] + (lo - out.rep_start[id]), hi - lo});
      }
  }
  if (rows > kRowMask || send_rows > kRowMask) throw std::invalid_argument("row count exceeds the row-code range");
  p.rows_local = static_cast<int>(rows);
  p.rows_send = static_cast<int>(send_rows);
}

}  // namespace moe
