// rope.cu — position-embedding correction and the generic Gradient Scaler.
//
// Tree Training's forward must "correct position embedding by aligning each element with its
// original position in the original trajectory": RoPE is a pointwise op whose
// Jacobian depends on the position m (Y = Rope(X, m)), so Eq. 23 (dY/dX identical in tree
// and per-branch packing) holds only if every token is rotated by its RESTORED position
// pos_i (tt_pack, R4) rather than its packed index.  The backward of a rotation is the rotation by
// the negative angle, dX = R(-m theta) dY, so the same kernel serves both directions.
//
// RoPE convention (reading R21; the paper names RoPE but not its variant): the "rotate-half" form
// used by Qwen-family models, over the whole head dim d:
//   theta_j = base^(-2j/d),  j < d/2;   a = pos * theta_j
//   y_j       = x_j cos a - x_{j+d/2} sin a
//   y_{j+d/2} = x_j sin a + x_{j+d/2} cos a
// The angle is formed and reduced mod 2 pi in fp64 (pos up to 2^31 times theta_0 = 1 would lose
// ~1e-3 rad in fp32), then cos / sin in fp32; x is read and written in the tensor's dtype
// (bf16: fp32 math, one RNE rounding).
//
// tt_restore_grad is the Gradient Scaler of P:549 ("insert a gradient scaling step before the
// backward propagation") for an arbitrary upstream gradient: row i of g is multiplied by its
// tree-scale (W_i when tt_pack_weights set real weights, else the integer leaf count w_i).  By the
// transitivity of Eqs. 17-21 every later pointwise / linear / attention backward then
// needs no further correction (tt_attn_bwd with restore = 0).
//
// Both kernels are HBM-bound: 2 x (row bytes) per row (read + write), coalesced 16-byte accesses.
#include <cmath>

#include "tt_internal.cuh"

namespace tt {
namespace {

constexpr int kRopeThreads = 256;
constexpr int kMaxHalf = 64;  // d <= 128

struct RopeArgs {
  int64_t N;
  int H, d;
  int inverse;
  const int32_t* pos;
  double inv_freq[kMaxHalf];  // base^(-2j/d), j < d/2, computed on the host in fp64
};

__device__ __forceinline__ void rope_angles(double pos, const double* invf, int j0, int cnt, float* c, float* s) {
  const double two_pi = 6.283185307179586476925286766559;
  for (int t = 0; t < cnt; ++t) {
    const double a = pos * invf[j0 + t];
    const double r = a - two_pi * rint(a * (1.0 / two_pi));  // in [-pi, pi]
    sincosf((float)r, &s[t], &c[t]);
  }
}

// One group of G = d/16 threads per (token, group of 4 heads): thread t of the group owns pairs j in
// [8t, 8t+8) (first half x[8t..8t+8) and second half x[d/2+8t..+8)), computes their 8 angles once
// and applies them to its 4 heads of the token.  All 8 16-byte loads of a thread are issued before
// any store (the head rows do not alias, but the compiler cannot know), so each thread keeps 128 B
// in flight: measured 0.77 of the HBM copy bandwidth with one head per load-store round trip
// (bench r1m next_f2), which is what this restructuring addresses.
constexpr int kRopeHeads = 4;
template <typename T>
__global__ void __launch_bounds__(kRopeThreads) rope_kernel(const RopeArgs a, T* __restrict__ x) {
  const int G = a.d / 16;
  const int HG = (a.H + kRopeHeads - 1) / kRopeHeads;
  const int64_t gid = ((int64_t)blockIdx.x * kRopeThreads + threadIdx.x);
  const int t = (int)(gid % G);
  const int64_t r = gid / G;
  const int hg = (int)(r % HG);
  const int64_t i = r / HG;
  if (i >= a.N) return;
  float c[8], s[8];
  rope_angles((double)a.pos[i], a.inv_freq, 8 * t, 8, c, s);
  if (a.inverse) {
#pragma unroll
    for (int u = 0; u < 8; ++u) s[u] = -s[u];
  }
  const int half = a.d / 2;
  const int h0 = hg * kRopeHeads;
  const int nh = min(kRopeHeads, a.H - h0);
  T* base = x + ((int64_t)i * a.H + h0) * a.d;
  if constexpr (sizeof(T) == 2) {
    uint4 A[kRopeHeads], B[kRopeHeads];
#pragma unroll
    for (int h = 0; h < kRopeHeads; ++h) {
      if (h < nh) {
        A[h] = *reinterpret_cast<const uint4*>(base + h * a.d + 8 * t);
        B[h] = *reinterpret_cast<const uint4*>(base + h * a.d + half + 8 * t);
      }
    }
#pragma unroll
    for (int h = 0; h < kRopeHeads; ++h) {
      if (h >= nh) continue;
      const uint32_t a4[4] = {A[h].x, A[h].y, A[h].z, A[h].w}, b4[4] = {B[h].x, B[h].y, B[h].z, B[h].w};
      uint32_t o1[4], o2[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float2 xa = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&a4[u]));
        const float2 xb = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&b4[u]));
        const float y1a = xa.x * c[2 * u] - xb.x * s[2 * u], y1b = xa.y * c[2 * u + 1] - xb.y * s[2 * u + 1];
        const float y2a = xa.x * s[2 * u] + xb.x * c[2 * u], y2b = xa.y * s[2 * u + 1] + xb.y * c[2 * u + 1];
        __nv_bfloat162 r1 = __floats2bfloat162_rn(y1a, y1b), r2 = __floats2bfloat162_rn(y2a, y2b);
        o1[u] = *reinterpret_cast<uint32_t*>(&r1);
        o2[u] = *reinterpret_cast<uint32_t*>(&r2);
      }
      *reinterpret_cast<uint4*>(base + h * a.d + 8 * t) = make_uint4(o1[0], o1[1], o1[2], o1[3]);
      *reinterpret_cast<uint4*>(base + h * a.d + half + 8 * t) = make_uint4(o2[0], o2[1], o2[2], o2[3]);
    }
  } else {
    for (int h = 0; h < nh; ++h) {
      float4* p1 = reinterpret_cast<float4*>(base + h * a.d + 8 * t);
      float4* p2 = reinterpret_cast<float4*>(base + h * a.d + half + 8 * t);
      const float4 A0 = p1[0], A1 = p1[1], B0 = p2[0], B1 = p2[1];
      const float xa[8] = {A0.x, A0.y, A0.z, A0.w, A1.x, A1.y, A1.z, A1.w};
      const float xb[8] = {B0.x, B0.y, B0.z, B0.w, B1.x, B1.y, B1.z, B1.w};
      float y1[8], y2[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        y1[k] = xa[k] * c[k] - xb[k] * s[k];
        y2[k] = xa[k] * s[k] + xb[k] * c[k];
      }
      p1[0] = make_float4(y1[0], y1[1], y1[2], y1[3]);
      p1[1] = make_float4(y1[4], y1[5], y1[6], y1[7]);
      p2[0] = make_float4(y2[0], y2[1], y2[2], y2[3]);
      p2[1] = make_float4(y2[4], y2[5], y2[6], y2[7]);
    }
  }
}

// g[i, :] *= scale_i   (16-byte vectors; row_elems % 8 == 0 for bf16, % 4 for fp32)
template <typename T>
__global__ void __launch_bounds__(256) restore_grad_kernel(T* __restrict__ g, int64_t N, int64_t row_vecs,
                                                           const int32_t* __restrict__ w, const float* __restrict__ wr) {
  const int64_t total = N * row_vecs;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < total; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = v / row_vecs;
    const float sc = wr ? wr[i] : (float)w[i];
    if constexpr (sizeof(T) == 2) {
      uint4* p = reinterpret_cast<uint4*>(g) + v;
      uint4 q = *p;
      uint32_t u4[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u4[u]));
        __nv_bfloat162 r = __floats2bfloat162_rn(f.x * sc, f.y * sc);
        u4[u] = *reinterpret_cast<uint32_t*>(&r);
      }
      *p = make_uint4(u4[0], u4[1], u4[2], u4[3]);
    } else {
      float4* p = reinterpret_cast<float4*>(g) + v;
      float4 q = *p;
      *p = make_float4(q.x * sc, q.y * sc, q.z * sc, q.w * sc);
    }
  }
}

}  // namespace

tt_status launch_rope(const tt_packed& pk, void* x, tt_dtype dt, int H, int d, double base, int inverse,
                      cudaStream_t st) {
  RopeArgs a;
  a.N = pk.n_tokens;
  a.H = H;
  a.d = d;
  a.inverse = inverse ? 1 : 0;
  a.pos = pk.pos;
  for (int j = 0; j < d / 2; ++j) a.inv_freq[j] = std::pow(base, -2.0 * j / d);
  const int64_t threads = a.N * ((H + kRopeHeads - 1) / kRopeHeads) * (d / 16);
  const unsigned grid = (unsigned)((threads + kRopeThreads - 1) / kRopeThreads);
  if (dt == TT_BF16)
    rope_kernel<__nv_bfloat16><<<grid, kRopeThreads, 0, st>>>(a, static_cast<__nv_bfloat16*>(x));
  else
    rope_kernel<float><<<grid, kRopeThreads, 0, st>>>(a, static_cast<float*>(x));
  count_launch();
  return check_launch("rope_kernel");
}

tt_status launch_restore_grad(const tt_packed& pk, void* g, tt_dtype dt, int64_t row_elems, cudaStream_t st) {
  const int64_t per = (dt == TT_BF16) ? 8 : 4;
  const int64_t row_vecs = row_elems / per;
  const int64_t total = pk.n_tokens * row_vecs;
  const unsigned grid = (unsigned)std::min<int64_t>((total + 255) / 256, 148 * 8);
  if (dt == TT_BF16)
    restore_grad_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(static_cast<__nv_bfloat16*>(g), pk.n_tokens, row_vecs,
                                                             pk.w, pk.wr);
  else
    restore_grad_kernel<float><<<grid, 256, 0, st>>>(static_cast<float*>(g), pk.n_tokens, row_vecs, pk.w, pk.wr);
  count_launch();
  return check_launch("restore_grad_kernel");
}

}  // namespace tt
