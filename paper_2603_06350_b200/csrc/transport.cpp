// transport.cpp — NcclTransport and CopyTransport (see transport.h).
#include "transport.h"

#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <iterator>
#include <map>
#include <mutex>
#include <string>

#include "ctx_internal.h"

namespace moe {

namespace {

class NcclTransport final : public Transport {
 public:
  explicit NcclTransport(ncclComm_t comm) : comm_(comm) {}
  void all_gather(const int32_t* mine, int32_t* all, size_t n, cudaStream_t s) override {
    g_nccl.check(g_nccl.AllGather(mine, all, n, ncclInt32, comm_, s), "ncclAllGather");
  }
  void exchange(const std::vector<Msg>& sends, const std::vector<Msg>& recvs, cudaStream_t s) override {
    g_nccl.check(g_nccl.GroupStart(), "ncclGroupStart");
    for (const Msg& m : sends) g_nccl.check(g_nccl.Send(m.buf, m.bytes, ncclUint8, m.peer, comm_, s), "ncclSend");
    for (const Msg& m : recvs) g_nccl.check(g_nccl.Recv(m.buf, m.bytes, ncclUint8, m.peer, comm_, s), "ncclRecv");
    g_nccl.check(g_nccl.GroupEnd(), "ncclGroupEnd");
  }

 private:
  ncclComm_t comm_;
};

// The ranks of one process that exchange together.
struct CopyHub {
  explicit CopyHub(int g) : G(g), ready(g, nullptr), done(g, nullptr) {}
  const int G;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long gen = 0;
  std::map<std::pair<int, int>, std::deque<std::pair<const void*, size_t>>> q;  // (src, dst) FIFO
  std::vector<cudaEvent_t> ready, done;  // per rank: its sends are written / its reads are done

  // all G ranks arrive before any leaves; a missing rank fails the call
  void barrier(uint64_t timeout_ns, int rank, const char* what) {
    std::unique_lock<std::mutex> l(mu);
    const long g = gen;
    if (++arrived == G) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return;
    }
    if (!cv.wait_for(l, std::chrono::nanoseconds(timeout_ns), [&] { return gen != g; })) {
      --arrived;
      throw Status(MOE_ESTATE, std::string("copy transport: rank ") + std::to_string(rank) + " timed out in " + what +
                                   " (ranks out of step?)");
    }
  }
};

std::mutex g_hubs_mu;
std::map<std::string, std::weak_ptr<CopyHub>> g_hubs;

std::shared_ptr<CopyHub> hub_for(const void* group, int G) {
  const std::string key(static_cast<const char*>(group), 128);
  std::lock_guard<std::mutex> l(g_hubs_mu);
  for (auto it = g_hubs.begin(); it != g_hubs.end();)  // groups whose ranks are all gone
    it = it->second.expired() && it->first != key ? g_hubs.erase(it) : std::next(it);
  auto h = g_hubs[key].lock();
  if (!h) {
    h = std::make_shared<CopyHub>(G);
    g_hubs[key] = h;
  }
  if (h->G != G) throw Status(MOE_EINVAL, "copy transport group used with two world sizes");
  return h;
}

class CopyTransport final : public Transport {
 public:
  CopyTransport(std::shared_ptr<CopyHub> hub, int rank, int device, uint64_t timeout_ns)
      : hub_(std::move(hub)), rank_(rank), device_(device), timeout_(timeout_ns) {
    CU_CHECK(cudaSetDevice(device_));
    CU_CHECK(cudaEventCreateWithFlags(&ready_, cudaEventDisableTiming));
    CU_CHECK(cudaEventCreateWithFlags(&done_, cudaEventDisableTiming));
  }
  ~CopyTransport() override {
    cudaEventDestroy(ready_);
    cudaEventDestroy(done_);
  }

  void all_gather(const int32_t* mine, int32_t* all, size_t n, cudaStream_t s) override {
    std::vector<Msg> sends, recvs;
    for (int p = 0; p < hub_->G; ++p) {
      if (p == rank_) continue;
      sends.push_back(Msg{const_cast<int32_t*>(mine), n * sizeof(int32_t), p});
      recvs.push_back(Msg{all + static_cast<size_t>(p) * n, n * sizeof(int32_t), p});
    }
    CU_CHECK(cudaMemcpyAsync(all + static_cast<size_t>(rank_) * n, mine, n * sizeof(int32_t),
                             cudaMemcpyDeviceToDevice, s));
    exchange(sends, recvs, s);
  }

  void exchange(const std::vector<Msg>& sends, const std::vector<Msg>& recvs, cudaStream_t s) override {
    CopyHub& h = *hub_;
    CU_CHECK(cudaEventRecord(ready_, s));  // my send rows are written once the stream gets here
    {
      std::lock_guard<std::mutex> l(h.mu);
      h.ready[rank_] = ready_;
      for (const Msg& m : sends) h.q[{rank_, m.peer}].emplace_back(m.buf, m.bytes);
    }
    h.barrier(timeout_, rank_, "the send rendezvous");
    for (const Msg& m : recvs) {
      std::pair<const void*, size_t> src;
      cudaEvent_t ev;
      {
        std::lock_guard<std::mutex> l(h.mu);
        auto& dq = h.q[{m.peer, rank_}];
        if (dq.empty() || dq.front().second != m.bytes)
          throw Status(MOE_ESTATE, "copy transport: rank " + std::to_string(rank_) + " expects " +
                                       std::to_string(m.bytes) + " bytes from rank " + std::to_string(m.peer) +
                                       (dq.empty() ? ", none sent" : ", got " + std::to_string(dq.front().second)));
        src = dq.front();
        dq.pop_front();
        ev = h.ready[m.peer];
      }
      CU_CHECK(cudaStreamWaitEvent(s, ev, 0));
      CU_CHECK(cudaMemcpyAsync(m.buf, src.first, m.bytes, cudaMemcpyDefault, s));
    }
    CU_CHECK(cudaEventRecord(done_, s));
    {
      std::lock_guard<std::mutex> l(h.mu);
      h.done[rank_] = done_;
    }
    h.barrier(timeout_, rank_, "the copy rendezvous");
    // my send buffers may be rewritten only after every reader's copies
    for (int p = 0; p < h.G; ++p)
      if (p != rank_) CU_CHECK(cudaStreamWaitEvent(s, h.done[p], 0));
    std::lock_guard<std::mutex> l(h.mu);  // every message I sent has been received
    for (const Msg& m : sends)
      if (!h.q[{rank_, m.peer}].empty())
        throw Status(MOE_ESTATE, "copy transport: rank " + std::to_string(m.peer) + " did not receive every "
                                 "message of rank " + std::to_string(rank_));
  }

 private:
  std::shared_ptr<CopyHub> hub_;
  int rank_, device_;
  uint64_t timeout_;
  cudaEvent_t ready_ = nullptr, done_ = nullptr;
};

}  // namespace

std::unique_ptr<Transport> make_nccl_transport(void* comm) {
  return std::make_unique<NcclTransport>(static_cast<ncclComm_t>(comm));
}

std::unique_ptr<Transport> make_copy_transport(const void* group, int G, int rank, int device, uint64_t timeout_ns) {
  if (!group) throw Status(MOE_EINVAL, "MOE_EXCHANGE_COPY needs a 128-byte group id (nccl_unique_id)");
  return std::make_unique<CopyTransport>(hub_for(group, G), rank, device, timeout_ns);
}

}  // namespace moe
