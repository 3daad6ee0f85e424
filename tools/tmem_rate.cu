// tmem_rate.cu — tcgen05.ld / tcgen05.st throughput microbenchmark (development tool, not product code).
// One CTA per SM; W warps (W/4 per TMEM lane quadrant) each load 32 lanes x 32 columns (4 KB) per
// tcgen05.ld.32x32b.x32, repeatedly, and we report bytes per SM clock.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2511_00413_b200/csrc \
//        tools/tmem_rate.cu -o tools/tmem_rate.bin -lcuda && tools/tmem_rate.bin
#include <cstdio>
#include <cuda_runtime.h>

#include "sm100_ptx.cuh"

using namespace tt::sm100;

constexpr int kIters = 512;

template <int MODE>  // 0: ld x32 + wait each, 1: 4 lds in flight then wait, 2: st x32 + wait each
__global__ void tmem_rate(unsigned long long* out, int nwarps) {
  __shared__ uint32_t tm_slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    tmem_alloc(&tm_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tm_slot + ((uint32_t)((warp & 3) * 32) << 16) + 32 * ((warp >> 2) & 3);
  uint32_t acc = 0;
  __syncthreads();
  const unsigned long long t0 = clock64();
  if (warp < nwarps) {
    for (int it = 0; it < kIters; ++it) {
      if constexpr (MODE == 0) {
        uint32_t v[32];
        tmem_ld32(tm + 128 * (it & 3), v);
        tmem_wait_ld();
#pragma unroll
        for (int u = 0; u < 32; ++u) acc += v[u];
      } else if constexpr (MODE == 1) {
        uint32_t a[32], b[32];
        tmem_ld32(tm, a);
        tmem_ld32(tm + 128, b);
        tmem_wait_ld();
#pragma unroll
        for (int u = 0; u < 32; ++u) acc += a[u] ^ b[u];
      } else {
        uint32_t v[32];
#pragma unroll
        for (int u = 0; u < 32; ++u) v[u] = acc + u;
        tmem_st32(tm + 128 * (it & 3), v);
        tmem_wait_st();
        acc += 1;
      }
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (acc == 0x12345678u) out[1023] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tm_slot, 512);
  }
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, int nwarps) {
  unsigned long long* d;
  cudaMalloc(&d, 1024 * 8);
  tmem_rate<MODE><<<148, 512>>>(d, nwarps);
  tmem_rate<MODE><<<148, 512>>>(d, nwarps);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < 148; ++i) s += h[i];
  s /= 148;
  const double per_op = (MODE == 1 ? 2.0 : 1.0) * 4096.0;  // bytes per warp per iteration
  printf("%-34s warps %2d %s cycles %.0f  -> %.1f B/clk/SM\n", name, nwarps, e == cudaSuccess ? "ok" : cudaGetErrorString(e), s,
         per_op * kIters * nwarps / s);
  cudaFree(d);
}

int main() {
  for (int w : {4, 8, 16}) run<0>("tcgen05.ld 32x32b.x32 + wait", w);
  for (int w : {4, 8, 16}) run<1>("2 x tcgen05.ld in flight + wait", w);
  for (int w : {4, 8, 16}) run<2>("tcgen05.st 32x32b.x32 + wait", w);
  return 0;
}
