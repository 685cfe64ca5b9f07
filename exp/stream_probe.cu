// Probe: HBM read rate of the gate's access pattern vs row-contiguous streaming
// (exp/, not product code).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ int4 ldnc(const void* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

// P1: gate mapping: CTA = 32 rows, warp (mt = w&1, ks = w>>1), lane (g, c): rows mt*16+g, +8; 16 B at f = ks*slice + it*32 + 8c
template <int U>
__global__ void __launch_bounds__(256) p1(const uint16_t* x, int T, int d, int* sink) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, c = lane & 3, mt = w & 1, ks = w >> 1;
  const int r0 = blockIdx.x * 32 + mt * 16 + g, r1 = r0 + 8;
  const int slice = d / 4;
  int acc = 0;
  for (int kb = ks * slice; kb < ks * slice + slice; kb += 32 * U) {
    int4 a[U], b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { a[u] = ldnc(x + (size_t)r0 * d + kb + 32 * u + 8 * c); b[u] = ldnc(x + (size_t)r1 * d + kb + 32 * u + 8 * c); }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += a[u].x ^ b[u].y ^ a[u].z ^ b[u].w;
  }
  if (acc == 0x12345) sink[0] = acc;
}

// P2: row-contiguous: CTA = 32 rows, warp w streams rows 4w..4w+3, lane 16 B chunks, U in flight
template <int U>
__global__ void __launch_bounds__(256) p2(const uint16_t* x, int T, int d, int* sink) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int acc = 0;
  for (int r = 0; r < 4; ++r) {
    const uint16_t* row = x + (size_t)(blockIdx.x * 32 + w * 4 + r) * d;
    for (int f = lane * 8; f < d; f += 256 * U) {
      int4 a[U];
#pragma unroll
      for (int u = 0; u < U; ++u) a[u] = ldnc(row + f + 256 * u);
#pragma unroll
      for (int u = 0; u < U; ++u) acc += a[u].x ^ a[u].w;
    }
  }
  if (acc == 0x12345) sink[0] = acc;
}

// P3: whole-CTA contiguous: the CTA's 256 KB block read as one stream (thread i reads chunk i, i+256, ...)
template <int U>
__global__ void __launch_bounds__(256) p3(const uint16_t* x, int T, int d, int* sink) {
  const int4* blk = reinterpret_cast<const int4*>(x + (size_t)blockIdx.x * 32 * d);
  const int n = 32 * d / 8;
  int acc = 0;
  for (int i = threadIdx.x; i < n; i += 256 * U) {
    int4 a[U];
#pragma unroll
    for (int u = 0; u < U; ++u) a[u] = ldnc(blk + i + 256 * u);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += a[u].x ^ a[u].w;
  }
  if (acc == 0x12345) sink[0] = acc;
}

template <class F>
float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) f();
  cudaEventRecord(a);
  for (int i = 0; i < 20; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms / 20;
}

int main() {
  const int T = 16384, d = 4096;
  uint16_t* x; int* sink; uint8_t* flush;
  cudaMalloc(&x, (size_t)T * d * 2); cudaMalloc(&sink, 4); cudaMalloc(&flush, 256 << 20);
  cudaMemset(x, 1, (size_t)T * d * 2);
  const double gb = (double)T * d * 2 / 1e9;
  auto run = [&](const char* name, auto kern) {
    float ms = timeit([&] { cudaMemsetAsync(flush, 0, 256 << 20); kern<<<T / 32, 256>>>(x, T, d, sink); });
    float fl = timeit([&] { cudaMemsetAsync(flush, 0, 256 << 20); });
    printf("%s: %.1f us  (%.2f TB/s)\n", name, (ms - fl) * 1e3, gb / ((ms - fl) * 1e-3) / 1e3);
  };
  run("P1 gate mapping U=1", p1<1>);
  run("P1 gate mapping U=2", p1<2>);
  run("P1 gate mapping U=4", p1<4>);
  run("P2 row-contiguous U=2", p2<2>);
  run("P2 row-contiguous U=4", p2<4>);
  run("P3 block-contiguous U=2", p3<2>);
  run("P3 block-contiguous U=4", p3<4>);
  run("P3 block-contiguous U=8", p3<8>);
  printf("err=%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
