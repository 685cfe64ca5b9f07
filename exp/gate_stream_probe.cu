// Probe (exp/, not product): the floor for streaming the cfg2 gate input
// (x = 16384 x 4096 bf16 = 134 MB) with TMA, no MMA / epilogue, one launch at a
// time after an L2 flush — the K1 kernel's access pattern (128-row x 64-feature
// boxes, BKS boxes per stage) at grid 128 (one 128-token tile per CTA) vs a
// stream-K split of the same k-block units over 148 CTAs, and 64-row tiles.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../paper_2603_06350_b200/csrc/kernels/sm100_ptx.cuh"

using namespace moe;

// units u = 0 .. n_units-1; unit = (tile = u / kb_per_tile, kb = u % kb_per_tile);
// CTA c streams units [c * n_units / grid, (c + 1) * n_units / grid)
__global__ void __launch_bounds__(128, 1) probe(const __grid_constant__ CUtensorMap tmx, int rows_per_tile, int kb_per_tile,
                                                int n_units, int bks, int stages, uint32_t stage_bytes, int* sink) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[16], empty[16];
  const int u0 = (int)((long long)blockIdx.x * n_units / gridDim.x);
  const int u1 = (int)((long long)(blockIdx.x + 1) * n_units / gridDim.x);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint64_t pol = policy_evict_first();
    int stage = 0; uint32_t phase = 0;
    for (int u = u0; u < u1; ++u) {
      if (u - u0 >= stages) mbar_wait(&empty[stage], phase ^ 1);
      const int t = u / kb_per_tile, kb = u % kb_per_tile;
      mbar_arrive_expect_tx(&full[stage], stage_bytes);
      for (int q = 0; q < bks; ++q)
        tma_load_2d_hint(smem + stage * stage_bytes + q * rows_per_tile * 128, &tmx, &full[stage], (kb * bks + q) * 64,
                         t * rows_per_tile, pol);
      if (++stage == stages) { stage = 0; phase ^= 1; }
    }
  } else if (threadIdx.x == 32) {
    int stage = 0; uint32_t phase = 0, acc = 0;
    for (int u = u0; u < u1; ++u) {
      mbar_wait(&full[stage], phase);
      acc += smem[stage * stage_bytes + (u & 511)];
      mbar_arrive(&empty[stage]);
      if (++stage == stages) { stage = 0; phase ^= 1; }
    }
    if (acc == 0x7fffffff) *sink = (int)acc;
  }
}

__global__ void flush(int4* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_int4(i, 0, 0, 0);
}
__global__ void empty_kernel() {}

int main() {
  const int T = 16384, d = 4096;
  const size_t bytes = (size_t)T * d * 2;
  void* x; int* sink; int4* fl;
  const size_t fl_n = (size_t)256 << 20 >> 4;  // 256 MB
  cudaMalloc(&x, bytes); cudaMalloc(&sink, 4); cudaMalloc(&fl, fl_n * 16);
  cudaMemset(x, 1, bytes);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                           const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                           CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                           CUtensorMapFloatOOBfill)>(fn);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  {
    std::vector<float> v;
    for (int i = 0; i < 20; ++i) {
      cudaEventRecord(a); empty_kernel<<<148, 128>>>(); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); v.push_back(ms * 1e3f);
    }
    std::sort(v.begin(), v.end());
    printf("empty kernel (events): median %.2f us\n", v[v.size() / 2]);
  }
  struct V { int rows, bks, stages, grid; };
  std::vector<V> vs = {{128, 2, 5, 128}, {128, 2, 5, 148}, {128, 1, 10, 148}, {128, 4, 2, 148}, {128, 2, 6, 148},
                       {64, 2, 10, 148}, {64, 4, 5, 148}, {64, 2, 10, 256}, {128, 2, 5, 256}, {64, 2, 6, 296},
                       {128, 1, 6, 296}, {256, 1, 5, 148}};
  for (const V& c : vs) {
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)T}, strides[1] = {(cuuint64_t)d * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)c.rows}, es[2] = {1, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const uint32_t stage_bytes = c.bks * c.rows * 128;
    const int kb_per_tile = d / (64 * c.bks), tiles = T / c.rows, n_units = tiles * kb_per_tile;
    const size_t smem = c.stages * (size_t)stage_bytes + 1024;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    std::vector<float> v;
    for (int i = 0; i < 25; ++i) {
      flush<<<592, 512>>>(fl, fl_n);
      cudaEventRecord(a);
      probe<<<c.grid, 128, smem>>>(m, c.rows, kb_per_tile, n_units, c.bks, c.stages, stage_bytes, sink);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (i >= 3) v.push_back(ms * 1e3f);
    }
    std::sort(v.begin(), v.end());
    const float med = v[v.size() / 2];
    printf("rows %3d bks %d stages %2d grid %3d smem %6zu: median %.2f us (min %.2f)  %.2f TB/s  (%s)\n", c.rows, c.bks,
           c.stages, c.grid, smem, med, v[0], bytes / (med * 1e-6) / 1e12, cudaGetErrorString(cudaGetLastError()));
  }
}
