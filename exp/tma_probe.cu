// Probe (exp/, not product): how fast can 148 persistent CTAs stream the decode
// GEMM1 weight tiles (64 experts x 11 n-tiles x [256 rows x 2048 cols] bf16,
// 128B-swizzled 256x64 TMA boxes, 4-stage ring) with no MMA / A / epilogue?
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../paper_2603_06350_b200/csrc/kernels/sm100_ptx.cuh"

using namespace moe;
constexpr int STAGES = 4, BK = 64, BN = 256;
constexpr uint32_t kB = BN * BK * 2;

__global__ void __launch_bounds__(192, 1) stream_b(const __grid_constant__ CUtensorMap tmB,
                                                   const __grid_constant__ CUtensorMap tmA, int a_rows, int tiles,
                                                   int n_tiles, int rows_per_slot, int num_kb, int stages, int* sink, int spin) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[8], empty[8], done;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(&done, 1);
    fence_barrier_init();
  }
  __syncthreads();
  const uint64_t pol = policy_evict_first();
  if (threadIdx.x == 0) {  // producer
    int stage = 0; uint32_t phase = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
      const int e = t / n_tiles, n = t % n_tiles;
      for (int kb = 0; kb < num_kb; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        mbar_arrive_expect_tx(&full[stage], kB + a_rows * BK * 2);
        tma_load_2d_hint(smem + stage * (kB + 16384), &tmB, &full[stage], kb * BK, e * rows_per_slot + n * BN, pol);
        if (a_rows) tma_load_2d(smem + stage * (kB + 16384) + kB, &tmA, &full[stage], kb * BK, (e % 16) * 128);
        if (++stage == stages) { stage = 0; phase ^= 1; }
      }
    }
  } else if (threadIdx.x == 32) {  // consumer
    int stage = 0; uint32_t phase = 0; int acc = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x)
      for (int kb = 0; kb < num_kb; ++kb) {
        mbar_wait(&full[stage], phase);
        acc += smem[stage * (kB + 16384) + (kb & 1023)];
        mbar_arrive(&empty[stage]);
        if (++stage == stages) { stage = 0; phase ^= 1; }
      }
    if (acc == 0x7fffffff) *sink = acc;
    mbar_arrive(&done);
  } else if (threadIdx.x >= 64 && spin) {  // idle warps waiting like K4's epilogue warps
    mbar_wait(&done, 0);
  }
}

int main() {
  const int E = 64, rows = 2816, d = 2048, n_tiles = rows / BN;  // 11
  const size_t bytes = (size_t)E * rows * d * 2;
  void* w; int* sink;
  cudaMalloc(&w, bytes); cudaMalloc(&sink, 4); cudaMemset(w, 1, bytes);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                           const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                           CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                           CUtensorMapFloatOOBfill)>(fn);
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)E * rows}, strides[1] = {(cuuint64_t)d * 2};
  cuuint32_t box[2] = {64, 256}, es[2] = {1, 1};
  enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int tiles = 62 * n_tiles;  // 62 active experts
  void* xa; cudaMalloc(&xa, (size_t)2048 * d * 2); cudaMemset(xa, 1, (size_t)2048 * d * 2);
  CUtensorMap ma32, ma128;
  cuuint64_t adims[2] = {(cuuint64_t)d, 2048};
  cuuint32_t abox32[2] = {64, 32}, abox128[2] = {64, 128};
  enc(&ma32, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, xa, adims, strides, abox32, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&ma128, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, xa, adims, strides, abox128, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  for (int spin : {0, 1}) for (int a_rows : {128})
  for (int stages : {4}) {
    const size_t smem = stages * (kB + 16384) + 1024;
    cudaFuncSetAttribute(stream_b, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int grid : {148}) {
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      for (int i = 0; i < 3; ++i) stream_b<<<grid, spin ? 192 : 64, smem>>>(m, a_rows == 32 ? ma32 : ma128, a_rows, tiles, n_tiles, rows, d / BK, stages, sink, spin);
      cudaEventRecord(a);
      for (int i = 0; i < 10; ++i) stream_b<<<grid, spin ? 192 : 64, smem>>>(m, a_rows == 32 ? ma32 : ma128, a_rows, tiles, n_tiles, rows, d / BK, stages, sink, spin);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
      const double gb = (double)tiles * BN * d * 2 / 1e9;
      printf("spin %d a_rows %d stages %d grid %d: %.1f us  %.2f TB/s  (%s)\n", spin, a_rows, stages, grid, ms * 1e3, gb / (ms * 1e-3) / 1e3,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
}
