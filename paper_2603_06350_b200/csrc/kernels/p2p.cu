// p2p.cu — K6 over peer memory (MOE_EXCHANGE_P2P): the counts all-gather and
// the flag protocol around the two row exchanges.
//
// Every rank exports ONE device slab (flags | counts | received rows xp |
// expert outputs yp) and maps every peer's slab (CUDA IPC across processes,
// plain pointers inside one process, NVLink peer access across devices).
// The row movement itself is fused into the existing kernels: K3 dispatch
// stores each token row straight into its final row of the DESTINATION
// rank's xp (row code target = that rank), and K5 combine loads expert
// outputs straight from the owning rank's yp — no send/return staging
// buffers, no copy kernels, no NCCL on the data path (PAPER.md:713's
// all-to-all).
//
// Flags: flags[kind][src] in the RECEIVER's slab, written by rank src with a
// system-scope release store of the forward's epoch (monotone, never reset);
// waiters use acquire loads.  The epoch lives in device memory: the counts
// kernel opens a forward by incrementing it and every later kernel of the
// forward reads it, so a captured CUDA graph replays with fresh epochs.
// Per forward (epoch n):
//   kCounts  src's gate histogram for n is readable       (before the gather)
//   kRows    src finished storing its rows into my xp     (before GEMM1)
//   kOutputs src's GEMM2 for n is done, its yp readable    (before combine)
// Reuse safety follows from stream order: rank h overwrites its yp (GEMM2,
// n+1) only after kRows(n+1) from every peer, which each peer signals after
// its combine(n) finished reading h's yp; a rank's xp is rewritten (dispatch,
// n+1) only after its owner's kOutputs(n), i.e. after its GEMM1(n) read it;
// counts(n+1) are written after combine(n), after every peer read counts(n).
//
// Waits are bounded (globaltimer): a stalled peer sets an error word in
// mapped host memory and the kernel exits, so a broken peer fails the call
// instead of hanging the GPU.
#include <cstdint>

#include "dispatch_plan.h"

namespace moe {

constexpr int kMaxRanks = 8;
enum { kFlagCounts = 0, kFlagRows = 1, kFlagOutputs = 2, kFlagKinds = 4 };

struct PeerSlabs {
  uint32_t* flags[kMaxRanks];       // each rank's flag block [kFlagKinds][kMaxRanks]
  const int32_t* counts[kMaxRanks];  // each rank's gate (+predictor) histogram
};

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// thread g < G: publish `epoch` in rank g's flags[kind][src]
__device__ __forceinline__ void signal_all(const PeerSlabs& peers, int G, int kind, int src, uint32_t epoch) {
  const int g = threadIdx.x;
  if (g < G) {
    __threadfence_system();
    st_release_sys(peers.flags[g] + kind * kMaxRanks + src, epoch);
  }
}

// thread g < G: wait until my flags[kind][g] reaches epoch (wrap-safe compare)
__device__ __forceinline__ void wait_all(const uint32_t* my_flags, int G, int kind, uint32_t epoch,
                                         uint64_t timeout_ns, int* err) {
  const int g = threadIdx.x;
  if (g >= G) return;
  const uint32_t* f = my_flags + kind * kMaxRanks + g;
  const uint64_t t0 = globaltimer();
  while (static_cast<int32_t>(ld_acquire_sys(f) - epoch) < 0) {
    if (globaltimer() - t0 > timeout_ns) {
      atomicCAS(err, 0, 1 + kind * kMaxRanks + g);
      return;
    }
    __nanosleep(64);
  }
}

__global__ void __launch_bounds__(32)
p2p_signal_kernel(const __grid_constant__ PeerSlabs peers, int G, int kind, int src, const uint32_t* epoch) {
  signal_all(peers, G, kind, src, *epoch);
}

__global__ void __launch_bounds__(32) p2p_wait_kernel(const uint32_t* my_flags, int G, int kind, const uint32_t* epoch,
                                                      uint64_t timeout_ns, int* err) {
  // GEMM1 (launched programmatically) may start streaming weights while we wait
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  wait_all(my_flags, G, kind, *epoch, timeout_ns, err);
}

// opens the forward (epoch + 1), then signal + wait + gather:
// counts_all[g][:] = rank g's histogram (stride ints)
__global__ void __launch_bounds__(256)
p2p_counts_kernel(const __grid_constant__ PeerSlabs peers, int G, int rank, int stride, uint32_t* epoch_dev,
                  uint64_t timeout_ns, int* err, int32_t* __restrict__ counts_all) {
  const uint32_t epoch = *epoch_dev + 1u;
  __syncthreads();
  if (threadIdx.x == 0) *epoch_dev = epoch;
  if (threadIdx.x < 32) {
    signal_all(peers, G, kFlagCounts, rank, epoch);
    wait_all(peers.flags[rank], G, kFlagCounts, epoch, timeout_ns, err);
  }
  __syncthreads();
  if (*reinterpret_cast<volatile int*>(err)) return;
  for (int i = threadIdx.x; i < G * stride; i += blockDim.x) {
    const int g = i / stride;
    counts_all[i] = __ldcv(peers.counts[g] + (i - g * stride));  // straight from the peer, no stale L1 line
  }
}

cudaError_t launch_p2p_signal(const PeerSlabs& peers, int G, int kind, int src, const uint32_t* epoch,
                              cudaStream_t s) {
  if (G > kMaxRanks) return cudaErrorInvalidValue;
  p2p_signal_kernel<<<1, 32, 0, s>>>(peers, G, kind, src, epoch);
  return cudaGetLastError();
}

cudaError_t launch_p2p_wait(const uint32_t* my_flags, int G, int kind, const uint32_t* epoch, uint64_t timeout_ns,
                            int* err, cudaStream_t s) {
  if (G > kMaxRanks) return cudaErrorInvalidValue;
  p2p_wait_kernel<<<1, 32, 0, s>>>(my_flags, G, kind, epoch, timeout_ns, err);
  return cudaGetLastError();
}

cudaError_t launch_p2p_counts(const PeerSlabs& peers, int G, int rank, int stride, uint32_t* epoch,
                              uint64_t timeout_ns, int* err, int32_t* counts_all, cudaStream_t s) {
  if (G > kMaxRanks) return cudaErrorInvalidValue;
  p2p_counts_kernel<<<1, 256, 0, s>>>(peers, G, rank, stride, epoch, timeout_ns, err, counts_all);
  return cudaGetLastError();
}

// Load every kernel of this file now (CUDA 12 loads kernels lazily on first
// launch, and a lazy load may wait for the whole context — including a
// peer-exchange kernel spinning on another rank that shares the context).
cudaError_t preload_p2p_kernels() {
  cudaFuncAttributes a;
  const void* fns[] = {reinterpret_cast<const void*>(p2p_signal_kernel),
                       reinterpret_cast<const void*>(p2p_wait_kernel),
                       reinterpret_cast<const void*>(p2p_counts_kernel)};
  for (const void* f : fns) {
    const cudaError_t e = cudaFuncGetAttributes(&a, f);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace moe
