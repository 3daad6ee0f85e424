// reduce.cu — HBM-bound helpers: the backward preprocess and the
// deterministic fp64 sum of squares used for the per-tree gradient-norm scalars (row a6).
#include "tt_internal.cuh"

namespace tt {
namespace {

template <typename T> __device__ __forceinline__ float ld_f(const T* p);
template <> __device__ __forceinline__ float ld_f<float>(const float* p) { return *p; }
template <> __device__ __forceinline__ float ld_f<__nv_bfloat16>(const __nv_bfloat16* p) { return __bfloat162float(*p); }

// D_i = dO_i . O_i per (token, head) (unweighted; the tree-scale enters in the main backward).
// One warp per row; bf16 rows of 128 are read as 8-byte vectors.  Optionally zeroes the fp32
// dQ accumulator row (the tcgen05 backward accumulates dQ with reductions).
template <typename T>
__global__ void __launch_bounds__(256) bwd_pre_kernel(const T* __restrict__ o, const T* __restrict__ dout, int64_t N,
                                                      int hq, int d, float* __restrict__ Dvec, float* __restrict__ dq_acc) {
  const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= N * hq) return;
  const int64_t i = row / hq;
  const int h = (int)(row % hq);
  const T* a = o + row * d;
  const T* b = dout + row * d;
  float s = 0.f;
  if constexpr (sizeof(T) == 2) {
    if (d == 128) {
      const uint2 va = reinterpret_cast<const uint2*>(a)[lane];
      const uint2 vb = reinterpret_cast<const uint2*>(b)[lane];
      const __nv_bfloat162* pa = reinterpret_cast<const __nv_bfloat162*>(&va);
      const __nv_bfloat162* pb = reinterpret_cast<const __nv_bfloat162*>(&vb);
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        float2 fa = __bfloat1622float2(pa[t]), fb = __bfloat1622float2(pb[t]);
        s = fmaf(fa.x, fb.x, s);
        s = fmaf(fa.y, fb.y, s);
      }
    } else {
      for (int c = lane; c < d; c += 32) s = fmaf(ld_f(a + c), ld_f(b + c), s);
    }
  } else {
    for (int c = lane; c < d; c += 32) s = fmaf(ld_f(a + c), ld_f(b + c), s);
  }
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (lane == 0) Dvec[(int64_t)h * N + i] = s;
  if (dq_acc) {
    float4* z = reinterpret_cast<float4*>(dq_acc + row * d);
    for (int c = lane; c < d / 4; c += 32) z[c] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// Tensor-core backward preprocess: per (token, head) -D_i = -dO_i . O_i, -LSE_i in log2 units, and
// per token the tree-scale as fp32 (w_i, or 1 without restoration), all laid out with the token
// dimension padded to Np (a multiple of 128) so the kernel can bulk-copy 64-row slices; padded rows
// get D = 0, LSE = 0, w = 0.  Also zeroes the fp32 dQ accumulator.
// 16 lanes per (token, head) row (16 bytes of O and of dO each), 8 rows per warp with all loads issued
// before the reductions (8 x 2 16-byte loads in flight per lane): the kernel is HBM-bound (reads O,
// dO, writes the zeroed fp32 dQ accumulator).
constexpr int kPreRowsPerWarp = 8;
__global__ void __launch_bounds__(256) bwd_pre_tc_kernel(const __nv_bfloat16* __restrict__ o,
                                                         const __nv_bfloat16* __restrict__ dout,
                                                         const float* __restrict__ lse, const int32_t* __restrict__ w,
                                                         const float* __restrict__ wr,
                                                         int restore, int fold, int64_t N, int64_t Np, int hq,
                                                         float* __restrict__ Dp, float* __restrict__ L2p,
                                                         float* __restrict__ wf, float* __restrict__ dq_acc) {
  const int lane = threadIdx.x & 31, half = lane >> 4, l16 = lane & 15;
  const int64_t row0 = ((int64_t)blockIdx.x * 8 + (threadIdx.x >> 5)) * kPreRowsPerWarp;  // row = i * hq + h
  const int64_t nrows = Np * hq, vrows = N * hq;
  uint4 va[kPreRowsPerWarp / 2], vb[kPreRowsPerWarp / 2];
#pragma unroll
  for (int k = 0; k < kPreRowsPerWarp / 2; ++k) {
    const int64_t row = row0 + 2 * k + half;
    if (row < vrows) {
      va[k] = reinterpret_cast<const uint4*>(o + row * 128)[l16];
      vb[k] = reinterpret_cast<const uint4*>(dout + row * 128)[l16];
    } else {
      va[k] = make_uint4(0, 0, 0, 0);
      vb[k] = va[k];
    }
  }
#pragma unroll
  for (int k = 0; k < kPreRowsPerWarp / 2; ++k) {
    const int64_t row = row0 + 2 * k + half;
    const uint32_t a4[4] = {va[k].x, va[k].y, va[k].z, va[k].w}, b4[4] = {vb[k].x, vb[k].y, vb[k].z, vb[k].w};
    float s = 0.f;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const float2 fa = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&a4[t]));
      const float2 fb = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&b4[t]));
      s = fmaf(fa.x, fb.x, s);
      s = fmaf(fa.y, fb.y, s);
    }
    for (int off = 8; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (row < vrows) {
      float4* z = reinterpret_cast<float4*>(dq_acc + row * 128) + 2 * l16;
      z[0] = make_float4(0.f, 0.f, 0.f, 0.f);
      z[1] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (l16 == 0 && row < nrows) {
      const int64_t i = row / hq;
      const int h = (int)(row % hq);
      Dp[(int64_t)h * Np + i] = -s;                                              // stored negated
      const float wv = i < N ? (restore ? (wr ? wr[i] : (float)w[i]) : 1.f) : 0.f;
      // stored negated; fold: + log2 w (w >= 0; w = 0 gives -inf, i.e. P w = 0)
      L2p[(int64_t)h * Np + i] = i < N ? -lse[(int64_t)h * N + i] * kLog2e + (fold ? log2f(wv) : 0.f) : 0.f;
      if (h == 0) wf[i] = wv;
    }
  }
}

// Sum of squares over up to 3 tensors in one launch: kSqnormBlocks fixed contiguous partitions per
// tensor (blockIdx.y = tensor), 16-byte vector loads (4 in flight per thread).  The squares of one
// vector are summed in fp32 (squares of bf16 values are exact in fp32; the 8-term fp32 sum has
// relative error <= 2^-21), vectors are accumulated in fp64, then fixed-order tree reductions —
// bitwise reproducible.
struct SqArgs {
  const void* x[3];
  int64_t n[3];
};

template <typename T>
__global__ void __launch_bounds__(256) sqnorm_partial_kernel(SqArgs a, double* __restrict__ part) {
  constexpr int E = 16 / sizeof(T);
  const int tsr = blockIdx.y;
  const T* x = static_cast<const T*>(a.x[tsr]);
  const int64_t n = a.n[tsr];
  const int64_t nv = n / E;
  const int64_t per = (nv + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = (int64_t)blockIdx.x * per;
  const int64_t b1 = imin64(nv, b0 + per);
  const uint4* xv = reinterpret_cast<const uint4*>(x);
  double s = 0.0;
  auto vsq = [&](const uint4& u) -> float {
    float r = 0.f;
    if constexpr (sizeof(T) == 2) {
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const float2 f = __bfloat1622float2(h[t]);
        r = fmaf(f.x, f.x, r);
        r = fmaf(f.y, f.y, r);
      }
    } else {
      const float* f = reinterpret_cast<const float*>(&u);
#pragma unroll
      for (int t = 0; t < 4; ++t) r = fmaf(f[t], f[t], r);
    }
    return r;
  };
  int64_t i = b0 + threadIdx.x;
  for (; i + 3 * blockDim.x < b1; i += 4 * blockDim.x) {
    const uint4 u0 = __ldg(xv + i), u1 = __ldg(xv + i + blockDim.x), u2 = __ldg(xv + i + 2 * blockDim.x),
                u3 = __ldg(xv + i + 3 * blockDim.x);
    s += (double)vsq(u0);
    s += (double)vsq(u1);
    s += (double)vsq(u2);
    s += (double)vsq(u3);
  }
  for (; i < b1; i += blockDim.x) s += (double)vsq(__ldg(xv + i));
  if (blockIdx.x == 0)
    for (int64_t t = nv * E + threadIdx.x; t < n; t += blockDim.x) {
      const double v = (double)ld_f(x + t);
      s = fma(v, v, s);
    }
  __shared__ double sh[256];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[(int64_t)tsr * gridDim.x + blockIdx.x] = sh[0];
}

__global__ void __launch_bounds__(256) sum_partials_kernel(const double* __restrict__ part, int n, double* __restrict__ out) {
  part += (int64_t)blockIdx.x * n;
  out += blockIdx.x;
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
  __shared__ double sh[256];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

}  // namespace

tt_status launch_bwd_pre(const void* o, const void* dout, tt_dtype dt, int64_t N, int hq, int d, float* Dvec,
                         float* dq_acc, cudaStream_t st) {
  const int64_t rows = N * hq;
  const unsigned blocks = (unsigned)((rows + 7) / 8);
  if (dt == TT_BF16)
    bwd_pre_kernel<__nv_bfloat16><<<blocks, 256, 0, st>>>((const __nv_bfloat16*)o, (const __nv_bfloat16*)dout, N, hq, d,
                                                          Dvec, dq_acc);
  else
    bwd_pre_kernel<float><<<blocks, 256, 0, st>>>((const float*)o, (const float*)dout, N, hq, d, Dvec, dq_acc);
  count_launch();
  return check_launch("bwd_pre_kernel");
}

tt_status launch_bwd_pre_tc(const void* o, const void* dout, const float* lse, const int32_t* w, const float* wr, int restore,
                            int fold, int64_t N, int64_t Np, int hq, float* Dp, float* L2p, float* wf, float* dq_acc,
                            cudaStream_t st) {
  const int64_t rows = Np * hq;
  bwd_pre_tc_kernel<<<(unsigned)((rows + 8 * kPreRowsPerWarp - 1) / (8 * kPreRowsPerWarp)), 256, 0, st>>>((const __nv_bfloat16*)o, (const __nv_bfloat16*)dout,
                                                               lse, w, wr, restore, fold, N, Np, hq, Dp, L2p, wf, dq_acc);
  count_launch();
  return check_launch("bwd_pre_tc_kernel");
}

tt_status launch_sqnorm(const void* const* xs, const int64_t* ns, int count, tt_dtype dt, double* out,
                        double* partials, cudaStream_t st) {
  SqArgs a{};
  for (int k = 0; k < count; ++k) { a.x[k] = xs[k]; a.n[k] = ns[k]; }
  const dim3 grid(kSqnormBlocks, count);
  if (dt == TT_BF16)
    sqnorm_partial_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(a, partials);
  else
    sqnorm_partial_kernel<float><<<grid, 256, 0, st>>>(a, partials);
  count_launch();
  tt_status s = check_launch("sqnorm_partial_kernel");
  if (s) return s;
  sum_partials_kernel<<<count, 256, 0, st>>>(partials, kSqnormBlocks, out);
  count_launch();
  return check_launch("sum_partials_kernel");
}

}  // namespace tt
