// transport.h — the message transport of the chunked expert exchange (K6,
// non-peer-memory modes).
//
// The exchange plan (host/exchange_plan.cpp) cuts every rank's rows into
// (peer, replica) chunks whose order is identical on both sides, so one step
// of the all-to-all is a grouped set of point-to-point messages matched per
// (source, destination) pair in issue order — NCCL's ncclGroupStart /
// ncclSend / ncclRecv / ncclGroupEnd semantics.  capi.cpp builds the message
// lists from the chunk lists once (stage_exchange) and hands them to a
// Transport:
//
//   NcclTransport  grouped ncclSend/ncclRecv + ncclAllGather (one process per
//                  GPU, NVLink/NVSwitch; MOE_EXCHANGE_NCCL)
//   CopyTransport  ranks of ONE process (threads, any devices): a host
//                  rendezvous per step, then every receiver pulls its messages
//                  with cudaMemcpyAsync (copy engines; peer copies between
//                  GPUs) after waiting on the sender's ready event, and no
//                  rank reuses a buffer before every reader's copy is done
//                  (MOE_EXCHANGE_COPY).  It is how the NCCL code path — chunk
//                  lists, message order, buffer offsets — runs with several
//                  ranks on the one-GPU boxes of this pool, and a transport
//                  for a single process driving several GPUs.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <memory>
#include <vector>

namespace moe {

struct Msg {
  void* buf;     // send: source rows; recv: destination rows (device)
  size_t bytes;
  int peer;
};

class Transport {
 public:
  virtual ~Transport() = default;
  // all[p * n .. (p+1) * n) = rank p's `mine` (int32, device)
  virtual void all_gather(const int32_t* mine, int32_t* all, size_t n, cudaStream_t s) = 0;
  // one grouped step: every send pairs with the peer's recv of the same
  // (source, destination) pair in issue order
  virtual void exchange(const std::vector<Msg>& sends, const std::vector<Msg>& recvs, cudaStream_t s) = 0;
};

std::unique_ptr<Transport> make_nccl_transport(void* comm /* ncclComm_t */);
// group: 128 bytes identifying the ranks of one process that exchange
// together (moe_ctx_desc.nccl_unique_id); timeout_ns bounds each rendezvous
std::unique_ptr<Transport> make_copy_transport(const void* group, int world_size, int rank, int device,
                                               uint64_t timeout_ns);

}  // namespace moe
