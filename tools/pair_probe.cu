// pair_probe.cu — development probe (not product code) for the tcgen05 cta_group::2 forms the CTA-pair
// backward needs, checked against host matmuls, plus their issue rates:
//   0  SS  M=256 N=64  K=64   A K-major SW128 (128 rows per CTA), B K-major SW128 (N-half per CTA)
//   1  TS  M=256 N=64  K=64   A from each CTA's TMEM (packed bf16), B as in 0
//   2  SS  M=128 N=64  K=128  A MN-major SW128 (64 M per CTA), B MN-major SW64 (32 N per CTA);
//      expected accumulator layout (CuTe tmem_frg_2sm, M_MMA = 64): lane m + 64 (n >= N/2), column n % (N/2)
//   3..6 timing: 4096 back-to-back MMAs of 3: SS M256 N64, 4: SS M128 N64 (form 2), 5: TS M256 N64,
//        6: SS M256 N128
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2511_00413_b200/csrc \
//        tools/pair_probe.cu -o /tmp/pair_probe && /tmp/pair_probe
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "sm100_ptx.cuh"

using namespace tt::sm100;

constexpr int kImg = 65536;

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mma_pair_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_pair_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a), "l"(b), "r"(id), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void commit_pair(uint64_t* bar) {
  asm volatile(
      "{\n.reg .pred e;\n.reg .b16 m;\nmov.b16 m, 3;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n}\n" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ uint64_t sdesc_l(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    probe(int test, const uint8_t* img, const uint32_t* tma, float* out, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const uint32_t rank = cta_rank();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint4* src = reinterpret_cast<const uint4*>(img + (size_t)rank * kImg);
  for (int i = threadIdx.x; i < kImg / 16; i += 128) reinterpret_cast<uint4*>(smem)[i] = src[i];
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tm = slot;
  const uint32_t tl = tm + ((uint32_t)(warp * 32) << 16);
  if (test == 1 || test == 5) {
    uint32_t v[32];
    for (int j = 0; j < 32; ++j) v[j] = tma[((size_t)rank * 128 + threadIdx.x) * 32 + j];
    tmem_st32(tl + 256, v);
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t sb = smem_u32(smem);
  if (rank == 0 && warp == 1) {
    const int reps = test >= 3 ? 4096 / 8 : 1;
    unsigned long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      if (test == 0 || test == 3 || test == 6) {
        const uint32_t id = idesc_bf16(256, test == 6 ? 128 : 64, 0, 0);
        const int nk = test == 0 ? 4 : 8;
        for (int kk = 0; kk < nk; ++kk)
          mma_pair_ss(tm, sdesc(sb + (kk & 3) * 32, 16, 1024), sdesc(sb + 16384 + (kk & 3) * 32, 16, 1024), id,
                      (r > 0 || kk > 0) ? 1u : 0u);
      } else if (test == 1 || test == 5) {
        const uint32_t id = idesc_bf16(256, 64, 0, 0);
        const int nk = test == 1 ? 4 : 8;
        for (int kk = 0; kk < nk; ++kk)
          mma_pair_ts(tm, tm + 256 + 8 * (kk & 3), sdesc(sb + 16384 + (kk & 3) * 32, 16, 1024), id,
                      (r > 0 || kk > 0) ? 1u : 0u);
      } else {  // 2, 4
        const uint32_t id = idesc_bf16(128, 64, 1, 1);
        for (int kk = 0; kk < 8; ++kk)
          mma_pair_ss(tm, sdesc_l(sb + kk * 2048, 16384, 1024, 2), sdesc_l(sb + 16384 + kk * 1024, 8192, 512, 4), id,
                      (r > 0 || kk > 0) ? 1u : 0u);
      }
    }
    commit_pair(&bar);
    mbar_wait(&bar, 0);
    unsigned long long t1 = clock64();
    if (lane == 0) cyc[0] = t1 - t0;
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  {
    uint32_t v[32];
    for (int h = 0; h < 2; ++h) {
      tmem_ld32(tl + 32 * h, v);
      tmem_wait_ld();
      for (int j = 0; j < 32; ++j)
        out[((size_t)rank * 128 + threadIdx.x) * 64 + 32 * h + j] = __uint_as_float(v[j]);
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tm) : "memory");
  }
}

static uint16_t bf(float x) {
  __nv_bfloat16 b = __float2bfloat16(x);
  uint16_t u;
  memcpy(&u, &b, 2);
  return u;
}
static void put(std::vector<uint8_t>& img, int cta, size_t off, float x) {
  uint16_t u = bf(x);
  memcpy(&img[(size_t)cta * kImg + off], &u, 2);
}
// K-major SW128, rows of 64 elements
static size_t kmaj128(size_t base, int row, int k) {
  return base + row * 128 + (size_t)(((((k * 2) >> 4) ^ (row & 7))) << 4) + ((k * 2) & 15);
}
// MN-major SW128: rows = k, 64 MN elements per row
static size_t mn128(size_t base, int mn, int k) {
  return base + (size_t)k * 128 + (size_t)(((((mn * 2) >> 4) ^ (k & 7))) << 4) + ((mn * 2) & 15);
}
// MN-major SW64: rows = k, 32 MN elements per row
static size_t mn64(size_t base, int mn, int k) {
  return base + (size_t)k * 64 + (size_t)(((((mn * 2) >> 4) ^ ((k >> 1) & 3))) << 4) + ((mn * 2) & 15);
}

int main() {
  uint8_t* d_img;
  uint32_t* d_tma;
  float* d_out;
  unsigned long long* d_cyc;
  cudaMalloc(&d_img, 2 * kImg);
  cudaMalloc(&d_tma, 2 * 128 * 32 * 4);
  cudaMalloc(&d_out, 2 * 128 * 64 * 4);
  cudaMalloc(&d_cyc, 8);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, kImg);
  srand(7);
  auto rnd = []() { return (float)((rand() % 17) - 8) / 8.f; };
  int fails = 0;
  for (int test = 0; test <= 6; ++test) {
    std::vector<uint8_t> img(2 * kImg, 0);
    std::vector<uint32_t> tma(2 * 128 * 32, 0);
    std::vector<float> expect(2 * 128 * 64, 0.f);
    if (test == 0 || test == 1 || test >= 3) {
      float A[2][128][64], B[128][64];
      for (int c = 0; c < 2; ++c)
        for (int l = 0; l < 128; ++l)
          for (int k = 0; k < 64; ++k) A[c][l][k] = rnd();
      for (int n = 0; n < 128; ++n)
        for (int k = 0; k < 64; ++k) B[n][k] = rnd();
      const int N = test == 6 ? 128 : 64;
      for (int c = 0; c < 2; ++c) {
        for (int l = 0; l < 128; ++l)
          for (int k = 0; k < 64; ++k) {
            put(img, c, kmaj128(0, l, k), A[c][l][k]);
            if (k % 2 == 0) tma[((size_t)c * 128 + l) * 32 + k / 2] = bf(A[c][l][k]) | ((uint32_t)bf(A[c][l][k + 1]) << 16);
          }
        for (int n = 0; n < N / 2; ++n)
          for (int k = 0; k < 64; ++k) put(img, c, kmaj128(16384, n, k), B[n + c * N / 2][k]);
        for (int l = 0; l < 128; ++l)
          for (int n = 0; n < 64; ++n) {
            float s = 0;
            for (int k = 0; k < 64; ++k) s += A[c][l][k] * B[n][k];
            expect[((size_t)c * 128 + l) * 64 + n] = s;
          }
      }
    } else {  // test 2
      float A[128][128], B[128][64];  // A[m][k], B[k][n]
      for (int m = 0; m < 128; ++m)
        for (int k = 0; k < 128; ++k) A[m][k] = rnd();
      for (int k = 0; k < 128; ++k)
        for (int n = 0; n < 64; ++n) B[k][n] = rnd();
      for (int c = 0; c < 2; ++c) {
        for (int m = 0; m < 64; ++m)
          for (int k = 0; k < 128; ++k) put(img, c, mn128(0, m, k), A[64 * c + m][k]);
        for (int n = 0; n < 32; ++n)
          for (int k = 0; k < 128; ++k) put(img, c, mn64(16384, n, k), B[k][32 * c + n]);
        for (int m = 0; m < 64; ++m)
          for (int n = 0; n < 64; ++n) {
            float s = 0;
            for (int k = 0; k < 128; ++k) s += A[64 * c + m][k] * B[k][n];
            const int lane = m + 64 * (n >= 32), col = n % 32;
            expect[((size_t)c * 128 + lane) * 64 + col] = s;
          }
      }
    }
    cudaMemcpy(d_img, img.data(), 2 * kImg, cudaMemcpyHostToDevice);
    cudaMemcpy(d_tma, tma.data(), tma.size() * 4, cudaMemcpyHostToDevice);
    cudaMemset(d_out, 0, 2 * 128 * 64 * 4);
    probe<<<2, 128, kImg>>>(test, d_img, d_tma, d_out, d_cyc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("test %d: CUDA error %s\n", test, cudaGetErrorString(e));
      return 1;
    }
    std::vector<float> out(2 * 128 * 64);
    unsigned long long cyc = 0;
    cudaMemcpy(out.data(), d_out, out.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(&cyc, d_cyc, 8, cudaMemcpyDeviceToHost);
    if (test <= 2) {
      const int ncol = test == 2 ? 32 : 64;
      int bad = 0;
      double maxerr = 0;
      for (int c = 0; c < 2; ++c)
        for (int l = 0; l < 128; ++l)
          for (int n = 0; n < ncol; ++n) {
            const size_t i = ((size_t)c * 128 + l) * 64 + n;
            const double err = fabs(out[i] - expect[i]);
            maxerr = err > maxerr ? err : maxerr;
            if (err > 1e-3) ++bad;
          }
      printf("test %d: %s (mismatches %d, max err %.3g)\n", test, bad ? "FAIL" : "ok", bad, maxerr);
      if (bad) {
        ++fails;
        for (int c = 0; c < 2; ++c)
          for (int l : {0, 1, 31, 63, 64, 65, 127}) {
            printf("  cta %d lane %3d got:", c, l);
            for (int n = 0; n < 6; ++n) printf(" %7.2f", out[((size_t)c * 128 + l) * 64 + n]);
            printf("   exp:");
            for (int n = 0; n < 6; ++n) printf(" %7.2f", expect[((size_t)c * 128 + l) * 64 + n]);
            printf("\n");
          }
      }
    } else {
      const char* name[] = {"", "", "", "SS M256 N64", "SS M128 N64 (MN A, SW64 B)", "TS M256 N64", "SS M256 N128"};
      const int M = test == 4 ? 128 : 256, N = test == 6 ? 128 : 64;
      const double per = (double)cyc / 4096.0;
      const double floor_cyc = (double)(M > 128 ? M : 128) * N / 512.0;
      printf("rate %-28s %8.2f cycles/MMA (floor %.1f) -> %.1f%% of the pair's tensor peak\n", name[test], per,
             floor_cyc, 100.0 * (double)M * N * 16 / (per * 8192.0));
    }
  }
  printf("%s\n", fails ? "PROBE FAILED" : "all layout checks passed");
  return fails ? 1 : 0;
}
