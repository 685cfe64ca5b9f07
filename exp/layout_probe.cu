// Probe (exp/, not product): does the DRAM layout of a K-major weight operand change
// how fast TMA streams it?  The decode GEMM1 weight stream (64 experts x 2816 rows x
// 2048 cols bf16 = 738 MB), 148 persistent CTAs, 256-row x 64-col boxes (32 KB), 4-stage
// ring, L2 flushed before every launch:
//   rowmajor: rows of 4 KB, a box = 256 row segments of 128 B, 4 KB apart (today's layout)
//   blocked : [k-block][row][64 cols] — a box is one contiguous 32 KB run (3D tensor map)
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../paper_2603_06350_b200/csrc/kernels/sm100_ptx.cuh"

using namespace moe;
constexpr int STAGES = 4, BK = 64, BN = 256;
constexpr uint32_t kB = BN * BK * 2;

__device__ __forceinline__ void tma_load_3d(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
      ::"r"(smem_u32(smem_dst)), "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}

template <bool BLOCKED>
__global__ void __launch_bounds__(64, 1) stream_w(const __grid_constant__ CUtensorMap tm, int tiles, int num_kb, int* sink) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[STAGES], empty[STAGES];
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int stage = 0; uint32_t phase = 0; int n = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x)
      for (int kb = 0; kb < num_kb; ++kb, ++n) {
        if (n >= STAGES) mbar_wait(&empty[stage], phase ^ 1);
        mbar_arrive_expect_tx(&full[stage], kB);
        if (BLOCKED) tma_load_3d(smem + stage * kB, &tm, &full[stage], 0, t * BN, kb);
        else tma_load_2d(smem + stage * kB, &tm, &full[stage], kb * BK, t * BN);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
  } else if (threadIdx.x == 32) {
    int stage = 0; uint32_t phase = 0; int acc = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x)
      for (int kb = 0; kb < num_kb; ++kb) {
        mbar_wait(&full[stage], phase);
        acc += smem[stage * kB + (kb & 1023)];
        mbar_arrive(&empty[stage]);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    if (acc == 0x7fffffff) *sink = acc;
  }
}

__global__ void flush(int4* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_int4(i, 0, 0, 0);
}

int main() {
  const int rows = 64 * 2816, K = 2048, num_kb = K / BK, tiles = rows / BN;
  const size_t bytes = (size_t)rows * K * 2;
  void* w; int* sink; int4* fl;
  const size_t fl_n = (size_t)256 << 20 >> 4;
  cudaMalloc(&w, bytes); cudaMalloc(&sink, 4); cudaMalloc(&fl, fl_n * 16);
  cudaMemset(w, 1, bytes);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                           const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                           CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                           CUtensorMapFloatOOBfill)>(fn);
  CUtensorMap m2, m3;
  {
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows}, strides[1] = {(cuuint64_t)K * 2};
    cuuint32_t box[2] = {64, BN}, es[2] = {1, 1};
    enc(&m2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  {
    cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)num_kb};
    cuuint64_t strides[2] = {128, (cuuint64_t)rows * 128};
    cuuint32_t box[3] = {64, BN, 1}, es[3] = {1, 1, 1};
    CUresult r = enc(&m3, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, w, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("3d map encode failed %d\n", (int)r);
  }
  const size_t smem = STAGES * kB + 1024;
  cudaFuncSetAttribute(stream_w<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(stream_w<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep)
    for (int blocked = 0; blocked < 2; ++blocked) {
      std::vector<float> v;
      for (int i = 0; i < 12; ++i) {
        flush<<<592, 512>>>(fl, fl_n);
        cudaEventRecord(a);
        if (blocked) stream_w<true><<<148, 64, smem>>>(m3, tiles, num_kb, sink);
        else stream_w<false><<<148, 64, smem>>>(m2, tiles, num_kb, sink);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (i >= 2) v.push_back(ms * 1e3f);
      }
      std::sort(v.begin(), v.end());
      printf("%s: median %.1f us (min %.1f)  %.2f TB/s  (%s)\n", blocked ? "blocked " : "rowmajor", v[v.size() / 2], v[0],
             bytes / (v[v.size() / 2] * 1e-6) / 1e12, cudaGetErrorString(cudaGetLastError()));
    }
}
