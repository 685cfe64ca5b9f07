#pragma once
#include <cstdint>
#include <vector>

#include "../kernels/dispatch_plan.h"

namespace moe {

struct Chunk {
  int peer;
  int replica;
  int64_t row_offset;
  int64_t rows;
};

struct HostPlan {
  DevPlan dev;
  std::vector<Chunk> sends;  // offsets into this rank's send buffer
  std::vector<Chunk> recvs;  // offsets into this rank's received-rows buffer
  std::vector<int64_t> rep_start, rep_size, seg_start;
  int64_t rows_local = 0, rows_send = 0;
};

// counts_all: [G][E]; R: [E]; gpu_of: [sum R] flattened (expert, ordinal).
// direct = false: remote rows go to this rank's send buffer (row-code target
// kSendTarget) for the NCCL / external exchange, described by sends/recvs.
// direct = true (peer-memory exchange): every row code names the destination
// rank and the row inside THAT rank's received-rows buffer, so dispatch
// stores each row straight into its final place on the owning GPU; no chunk
// lists, rows_send counts the rows that leave this GPU.
void build_exchange_plan(int G, int rank, int E, const int64_t* counts_all, const int32_t* R,
                         const int32_t* gpu_of, HostPlan& out, bool direct = false);

}  // namespace moe
