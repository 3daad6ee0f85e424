// mma_rate.cu — tcgen05.mma issue-rate microbenchmark (development tool, not product code).
// One CTA per SM issues back-to-back kind::f16 MMAs of one shape/operand source and times them
// with clock64, to measure how shared-memory operand reads pace each shape on sm_100a:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2511_00413_b200/csrc \
//        tools/mma_rate.cu -o /tmp/mma_rate -lcuda && /tmp/mma_rate
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>

#include "sm100_ptx.cuh"

using namespace tt::sm100;

constexpr int kIters = 2048;  // MMA instructions (K = 16 each) per measurement

// variant: 0 SS N64, 1 SS N128, 2 SS N256, 3 TS N64, 4 TS N128, 5 TS N256,
//          6 SS N64 A MN-major (dQ^T shape), 7 SS N128 with concurrent LDS traffic
template <int V>
__global__ void __launch_bounds__(128, 1) mma_rate(unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tm_slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u ^ (i * 2654435761u & 0x00ff00ffu);
  if (warp == 0) {
    tmem_alloc(&tm_slot, 512);
    tmem_relinquish();
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tm_slot;
  constexpr int N = (V == 0 || V == 3 || V == 6) ? 64 : (V == 1 || V == 4 || V == 7) ? 128 : 256;
  constexpr bool ts = (V >= 3 && V <= 5);
  const uint32_t a_s = smem_u32(smem), b_s = a_s + 32 * 1024;
  const uint32_t id = idesc_bf16(128, N, V == 6 ? 1 : 0, 0);
  unsigned long long t0 = 0, t1 = 0;
  if (warp == 1) {
    t0 = clock64();
    for (int it = 0; it < kIters / 8; ++it) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t offa = (kk >> 2) * 16384 + (kk & 3) * 32;
        const uint32_t offb = (kk >> 2) * (N * 128) + (kk & 3) * 32;
        if constexpr (ts)
          mma_ts_w(tm, tm + 256 + 8 * kk, sdesc(b_s + offb, 16, 1024), id, 1u);
        else if constexpr (V == 6)
          mma_ss_w(tm, sdesc(a_s + kk * 2048, 16384, 1024), sdesc(b_s + offb, 16, 1024), id, 1u);
        else
          mma_ss_w(tm, sdesc(a_s + offa, 16, 1024), sdesc(b_s + offb, 16, 1024), id, 1u);
      }
    }
    mma_commit_w(&bar);
    mbar_wait(&bar, 0);
    t1 = clock64();
  } else if (V == 7 && warp >= 2) {
    // concurrent shared-memory reads (LDS.128) by two warps while the MMAs run
    uint4 acc = make_uint4(0, 0, 0, 0);
    const uint4* p = reinterpret_cast<const uint4*>(smem + 64 * 1024);
    for (int i = 0; i < kIters * 4; ++i) {
      uint4 x = p[(i * 32 + (threadIdx.x & 31)) & 2047];
      acc.x ^= x.x; acc.y += x.y;
    }
    if (acc.x == 0x12345 && acc.y == 7) out[1000] = 1;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tm, 512);
  }
  if (threadIdx.x == 32) out[blockIdx.x] = t1 - t0;
}

template <int V>
void run(const char* name) {
  unsigned long long* d;
  cudaMalloc(&d, 1024 * 8 + 8);
  cudaFuncSetAttribute(mma_rate<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  mma_rate<V><<<148, 128, 100 * 1024>>>(d);
  mma_rate<V><<<148, 128, 100 * 1024>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < 148; ++i) s += h[i];
  s /= 148;
  const int N = (V == 0 || V == 3 || V == 6) ? 64 : (V == 1 || V == 4 || V == 7) ? 128 : 256;
  const double cyc = s / kIters;
  const double floor = 128.0 * N / 256.0;
  printf("%-28s %s  cycles/MMA(K16) %.1f  floor %.0f  -> %.2f of tensor floor, %.0f FLOP/clk/SM\n", name,
         e == cudaSuccess ? "ok " : cudaGetErrorString(e), cyc, floor, floor / cyc, 128.0 * N * 16 * 2 / cyc);
  cudaFree(d);
}

int main() {
  run<0>("SS M128 N64 (K-major)");
  run<1>("SS M128 N128");
  run<2>("SS M128 N256");
  run<3>("TS M128 N64 (A in TMEM)");
  run<4>("TS M128 N128");
  run<5>("TS M128 N256");
  run<6>("SS M128 N64, A MN-major");
  run<7>("SS M128 N128 + LDS traffic");
  return 0;
}
