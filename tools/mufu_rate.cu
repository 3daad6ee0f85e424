// MUFU exp2 throughput on sm_100a: ex2.approx.ftz.f32 vs ex2.approx.f16x2 vs ex2.approx.ftz.bf16x2
// (results per SM per clock, all SMs busy, 8 independent chains per thread).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mufu_rate tools/mufu_rate.cu && ./mufu_rate
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_bf16.h>

template <int MODE>
__global__ void k(float* out, int iters, long long* cyc) {
  uint32_t v[8];
  for (int i = 0; i < 8; ++i) v[i] = 0x3c003c00u ^ (threadIdx.x + i);  // small fp16 / bf16 / f32 bit patterns
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) {
        float x = __uint_as_float((v[i] & 0x807fffffu) | 0x3e000000u), y;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
        v[i] = __float_as_uint(y) ^ it;
      } else if (MODE == 1) {
        uint32_t y;
        asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(v[i] & 0xb3ffb3ffu));
        v[i] = y ^ it;
      } else if (MODE == 2) {
        uint32_t y;
        asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(v[i] & 0xbe7fbe7fu));
        v[i] = y ^ it;
      } else if (MODE == 3) {
        // F2FP: two fp32 -> packed bf16x2 (RNE)
        uint32_t y;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(y) : "f"(__uint_as_float(v[i])), "f"(__uint_as_float(v[i] ^ 0x1234u)));
        v[i] = y ^ it;
      } else if (MODE == 4) {
        // the same rounding on the integer pipe: (x + 0x7fff + ((x >> 16) & 1)) >> 16, two values, PRMT
        const uint32_t a = v[i], b = v[i] ^ 0x1234u;
        const uint32_t ra = a + 0x7fffu + ((a >> 16) & 1u), rb = b + 0x7fffu + ((b >> 16) & 1u);
        uint32_t y;
        asm volatile("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(y) : "r"(ra), "r"(rb));
        v[i] = y ^ it;
      } else {
        // f32x2 FMA (FFMA2) for reference
        float2 x = make_float2(__uint_as_float(v[i] & 0x3fffffffu), __uint_as_float((v[i] ^ 1) & 0x3fffffffu));
        float2 y;
        asm volatile("{\n.reg .b64 ra, rd;\nmov.b64 ra, {%2, %3};\nfma.rn.f32x2 rd, ra, ra, ra;\nmov.b64 {%0, %1}, rd;\n}" : "=f"(y.x), "=f"(y.y) : "f"(x.x), "f"(x.y));
        v[i] = __float_as_uint(y.x) ^ __float_as_uint(y.y) ^ it;
      }
    }
  }
  long long t1 = clock64();
  uint32_t acc = 0;
  for (int i = 0; i < 8; ++i) acc ^= v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 4 * 1024 * sizeof(float));
  cudaMalloc(&cyc, sizeof(long long));
  const int iters = 4096, threads = 1024, blocks = 148 * 2;
  const char* names[6] = {"ex2.approx.ftz.f32", "ex2.approx.f16x2", "ex2.approx.ftz.bf16x2", "cvt.rn.bf16x2.f32 (F2FP)",
                          "bf16 RNE on the integer pipe", "fma.rn.f32x2 (FFMA2)"};
  for (int mode = 0; mode < 6; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      if (mode == 0) k<0><<<blocks, threads>>>(out, iters, cyc);
      if (mode == 1) k<1><<<blocks, threads>>>(out, iters, cyc);
      if (mode == 2) k<2><<<blocks, threads>>>(out, iters, cyc);
      if (mode == 3) k<3><<<blocks, threads>>>(out, iters, cyc);
      if (mode == 4) k<4><<<blocks, threads>>>(out, iters, cyc);
      if (mode == 5) k<5><<<blocks, threads>>>(out, iters, cyc);
      cudaDeviceSynchronize();
    }
    long long c = 0;
    cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
    // per SM: 2 blocks x 1024 threads x iters x 8 instructions; values per instruction: 1 (f32) or 2
    const double insts = 2.0 * threads * iters * 8;
    const double vals = insts * (mode == 0 ? 1 : 2);  // values per instruction (F2FP / FFMA2 / int: 2)
    printf("%-24s %.2f instr/clk/SM  %.2f values/clk/SM  (%lld cycles)\n", names[mode], insts / c, vals / c, c);
  }
  return 0;
}
