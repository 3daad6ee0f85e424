// attn_simt.cu — SIMT (CUDA-core, fp32 arithmetic) tree-masked attention: the "test mode" of
// DESIGN.md R13.  tcgen05 has no fp32 kind and kind::tf32 cannot meet 1e-4, so fp32 I/O runs
// here; bf16 at d=64 also runs here.  (bf16 at d=128 runs on the tcgen05 kernels.)
//
// The kernels consume exactly the pack metadata the tensor-core kernels use: the forward walks
// the per-q-block tile list (empty tiles skipped, full tiles unmasked, partial tiles masked with
// j <= i < E_j), the dK/dV kernel walks the contiguous query range [j, E_j) of each key.
//
// Forward (Eq. 1):  online softmax in the log2 domain, LSE written in natural log.
// Backward (Eqs. 2, 20-21; App. B of SURVEY): omega_i = w_i when restoring, P recomputed from LSE,
//   dS_ij = omega_i P_ij (dO_i.v_j - D_i); dQ kernel (query-stationary) and dK/dV kernel
//   (key-stationary, summing the q heads of the kv group) — no atomics, deterministic.
#include "tt_internal.cuh"

namespace tt {
namespace {

template <typename T> __device__ __forceinline__ float to_f(T x);
template <> __device__ __forceinline__ float to_f<float>(float x) { return x; }
template <> __device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }
template <typename T> __device__ __forceinline__ T from_f(float x);
template <> __device__ __forceinline__ float from_f<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }

__device__ __forceinline__ float warp_max(float v) {
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

constexpr int kRows = 64;   // query rows (fwd / dq) or keys (dkdv) per CTA
constexpr int kChunk = 32;  // keys (fwd / dq) or queries (dkdv) staged per step
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kPerWarp = kRows / kWarps;  // 8

struct PackView {
  int64_t N;
  const int32_t* w;
  const float* wr;  // real-valued tree-scale (NEXT-f4) or null
  const int32_t* E;
  const int32_t* kmaxE;
  const int32_t* fwd_cnt;
  const int32_t* fwd_list;
};

// ---------------------------------------------------------------------------------------------
// forward
// ---------------------------------------------------------------------------------------------
template <typename T, int D>
__global__ void __launch_bounds__(kThreads) simt_fwd_kernel(PackView pv, const T* __restrict__ q, const T* __restrict__ k,
                                                            const T* __restrict__ v, int hq, int hkv, float scale_log2,
                                                            T* __restrict__ o, float* __restrict__ lse) {
  constexpr int DP = D + 1;
  constexpr int NC = D / 32;
  extern __shared__ float smem[];
  float* sQ = smem;                 // [kRows][D]
  float* sK = sQ + kRows * D;       // [kChunk][DP]
  float* sV = sK + kChunk * DP;     // [kChunk][D]
  float* sP = sV + kChunk * D;      // [kWarps][32]
  int* sE = reinterpret_cast<int*>(sP + kWarps * 32);

  const int64_t N = pv.N;
  const int qb = blockIdx.x >> 1;
  const int64_t r0 = (int64_t)qb * kBlock + (blockIdx.x & 1) * kRows;
  if (r0 >= N) return;
  const int h = blockIdx.y;
  const int hk = h / (hq / hkv);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  for (int idx = tid; idx < kRows * D; idx += kThreads) {
    const int r = idx / D, c = idx % D;
    const int64_t i = r0 + r;
    sQ[idx] = i < N ? to_f(q[(i * hq + h) * D + c]) : 0.f;
  }
  float m[kPerWarp], l[kPerWarp], acc[kPerWarp][NC];
#pragma unroll
  for (int rr = 0; rr < kPerWarp; ++rr) {
    m[rr] = -INFINITY;
    l[rr] = 0.f;
#pragma unroll
    for (int cc = 0; cc < NC; ++cc) acc[rr][cc] = 0.f;
  }
  const int cnt = pv.fwd_cnt[qb];
  const int32_t* list = pv.fwd_list + tri_off(qb);
  for (int t = 0; t < cnt; ++t) {
    const int32_t ent = list[t];
    const int kb = ent & kKbMask;
    const bool full = (ent >> kClsShift) == kClsFull;
    for (int ch = 0; ch < kBlock / kChunk; ++ch) {
      const int64_t j0 = (int64_t)kb * kBlock + ch * kChunk;
      if (j0 >= N) break;
      if (j0 > r0 + kRows - 1) break;  // keys beyond the last row are never allowed (j <= i)
      __syncthreads();
      for (int idx = tid; idx < kChunk * D; idx += kThreads) {
        const int jj = idx / D, c = idx % D;
        const int64_t j = j0 + jj;
        const bool in = j < N;
        sK[jj * DP + c] = in ? to_f(k[(j * hkv + hk) * D + c]) : 0.f;
        sV[jj * D + c] = in ? to_f(v[(j * hkv + hk) * D + c]) : 0.f;
      }
      if (tid < kChunk) sE[tid] = (j0 + tid < N) ? pv.E[j0 + tid] : -1;
      __syncthreads();
      const int64_t j = j0 + lane;
#pragma unroll
      for (int rr = 0; rr < kPerWarp; ++rr) {
        const int r = warp * kPerWarp + rr;
        const int64_t i = r0 + r;
        if (i >= N) continue;
        float s = 0.f;
#pragma unroll 8
        for (int c = 0; c < D; ++c) s = fmaf(sQ[r * D + c], sK[lane * DP + c], s);
        s *= scale_log2;
        const bool ok = (j < N) && (full ? (j <= i) : (j <= i && i < (int64_t)sE[lane]));
        s = ok ? s : -INFINITY;
        const float cm = warp_max(s);
        if (cm == -INFINITY) continue;
        const float mn = fmaxf(m[rr], cm);
        const float corr = exp2f(m[rr] - mn);
        const float p = exp2f(s - mn);
        l[rr] = l[rr] * corr + warp_sum(p);
        m[rr] = mn;
        sP[warp * 32 + lane] = p;
        __syncwarp();
#pragma unroll
        for (int cc = 0; cc < NC; ++cc) {
          float a = acc[rr][cc] * corr;
          const int c = lane + 32 * cc;
#pragma unroll 8
          for (int jj = 0; jj < kChunk; ++jj) a = fmaf(sP[warp * 32 + jj], sV[jj * D + c], a);
          acc[rr][cc] = a;
        }
        __syncwarp();
      }
    }
  }
#pragma unroll
  for (int rr = 0; rr < kPerWarp; ++rr) {
    const int64_t i = r0 + warp * kPerWarp + rr;
    if (i >= N) continue;
    const float inv = 1.f / l[rr];
#pragma unroll
    for (int cc = 0; cc < NC; ++cc) o[(i * hq + h) * D + lane + 32 * cc] = from_f<T>(acc[rr][cc] * inv);
    if (lane == 0) lse[(int64_t)h * N + i] = (m[rr] + log2f(l[rr])) * kLn2;
  }
}

// ---------------------------------------------------------------------------------------------
// backward: dQ (query-stationary)
// ---------------------------------------------------------------------------------------------
template <typename T, int D>
__global__ void __launch_bounds__(kThreads) simt_dq_kernel(PackView pv, const T* __restrict__ q, const T* __restrict__ k,
                                                           const T* __restrict__ v, const float* __restrict__ lse,
                                                           const float* __restrict__ Dvec, const T* __restrict__ dout,
                                                           int restore, int hq, int hkv, float scale, float scale_log2,
                                                           T* __restrict__ dq) {
  constexpr int DP = D + 1;
  constexpr int NC = D / 32;
  extern __shared__ float smem[];
  float* sQ = smem;                   // [kRows][D]
  float* sG = sQ + kRows * D;         // [kRows][D]   dO rows
  float* sK = sG + kRows * D;         // [kChunk][DP]
  float* sV = sK + kChunk * DP;       // [kChunk][DP]
  float* sS = sV + kChunk * DP;       // [kWarps][32] dS
  int* sE = reinterpret_cast<int*>(sS + kWarps * 32);

  const int64_t N = pv.N;
  const int qb = blockIdx.x >> 1;
  const int64_t r0 = (int64_t)qb * kBlock + (blockIdx.x & 1) * kRows;
  if (r0 >= N) return;
  const int h = blockIdx.y;
  const int hk = h / (hq / hkv);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int idx = tid; idx < kRows * D; idx += kThreads) {
    const int r = idx / D, c = idx % D;
    const int64_t i = r0 + r;
    sQ[idx] = i < N ? to_f(q[(i * hq + h) * D + c]) : 0.f;
    sG[idx] = i < N ? to_f(dout[(i * hq + h) * D + c]) : 0.f;
  }
  float lse2[kPerWarp], Di[kPerWarp], om[kPerWarp], acc[kPerWarp][NC];
#pragma unroll
  for (int rr = 0; rr < kPerWarp; ++rr) {
    const int64_t i = r0 + warp * kPerWarp + rr;
    const bool in = i < N;
    lse2[rr] = in ? lse[(int64_t)h * N + i] * kLog2e : 0.f;
    Di[rr] = in ? Dvec[(int64_t)h * N + i] : 0.f;
    om[rr] = (in && restore) ? (pv.wr ? pv.wr[i] : (float)pv.w[i]) : 1.f;
#pragma unroll
    for (int cc = 0; cc < NC; ++cc) acc[rr][cc] = 0.f;
  }
  const int cnt = pv.fwd_cnt[qb];
  const int32_t* list = pv.fwd_list + tri_off(qb);
  for (int t = 0; t < cnt; ++t) {
    const int32_t ent = list[t];
    const int kb = ent & kKbMask;
    const bool full = (ent >> kClsShift) == kClsFull;
    for (int ch = 0; ch < kBlock / kChunk; ++ch) {
      const int64_t j0 = (int64_t)kb * kBlock + ch * kChunk;
      if (j0 >= N || j0 > r0 + kRows - 1) break;
      __syncthreads();
      for (int idx = tid; idx < kChunk * D; idx += kThreads) {
        const int jj = idx / D, c = idx % D;
        const int64_t j = j0 + jj;
        const bool in = j < N;
        sK[jj * DP + c] = in ? to_f(k[(j * hkv + hk) * D + c]) : 0.f;
        sV[jj * DP + c] = in ? to_f(v[(j * hkv + hk) * D + c]) : 0.f;
      }
      if (tid < kChunk) sE[tid] = (j0 + tid < N) ? pv.E[j0 + tid] : -1;
      __syncthreads();
      const int64_t j = j0 + lane;
#pragma unroll
      for (int rr = 0; rr < kPerWarp; ++rr) {
        const int r = warp * kPerWarp + rr;
        const int64_t i = r0 + r;
        if (i >= N) continue;
        float s = 0.f, dp = 0.f;
#pragma unroll 8
        for (int c = 0; c < D; ++c) {
          s = fmaf(sQ[r * D + c], sK[lane * DP + c], s);
          dp = fmaf(sG[r * D + c], sV[lane * DP + c], dp);
        }
        const bool ok = (j < N) && (full ? (j <= i) : (j <= i && i < (int64_t)sE[lane]));
        const float p = ok ? exp2f(s * scale_log2 - lse2[rr]) : 0.f;
        const float ds = om[rr] * p * (dp - Di[rr]);
        sS[warp * 32 + lane] = ds;
        __syncwarp();
#pragma unroll
        for (int cc = 0; cc < NC; ++cc) {
          const int c = lane + 32 * cc;
          float a = acc[rr][cc];
#pragma unroll 8
          for (int jj = 0; jj < kChunk; ++jj) a = fmaf(sS[warp * 32 + jj], sK[jj * DP + c], a);
          acc[rr][cc] = a;
        }
        __syncwarp();
      }
    }
  }
#pragma unroll
  for (int rr = 0; rr < kPerWarp; ++rr) {
    const int64_t i = r0 + warp * kPerWarp + rr;
    if (i >= N) continue;
#pragma unroll
    for (int cc = 0; cc < NC; ++cc) dq[(i * hq + h) * D + lane + 32 * cc] = from_f<T>(acc[rr][cc] * scale);
  }
}

// ---------------------------------------------------------------------------------------------
// backward: dK / dV (key-stationary; the queries of key j are the contiguous range [j, E_j))
// ---------------------------------------------------------------------------------------------
template <typename T, int D>
__global__ void __launch_bounds__(kThreads) simt_dkdv_kernel(PackView pv, const T* __restrict__ q, const T* __restrict__ k,
                                                             const T* __restrict__ v, const float* __restrict__ lse,
                                                             const float* __restrict__ Dvec, const T* __restrict__ dout,
                                                             int restore, int hq, int hkv, float scale, float scale_log2,
                                                             T* __restrict__ dk, T* __restrict__ dv) {
  constexpr int DP = D + 1;
  constexpr int NC = D / 32;
  extern __shared__ float smem[];
  float* sK = smem;                   // [kRows][D]
  float* sV = sK + kRows * D;         // [kRows][D]
  float* sQ = sV + kRows * D;         // [kChunk][DP]
  float* sG = sQ + kChunk * DP;       // [kChunk][DP]
  float* sL = sG + kChunk * DP;       // [kChunk] lse (log2)
  float* sD = sL + kChunk;            // [kChunk]
  float* sW = sD + kChunk;            // [kChunk]
  float* sPW = sW + kChunk;           // [kWarps][32]
  float* sS = sPW + kWarps * 32;      // [kWarps][32]
  int* sE = reinterpret_cast<int*>(sS + kWarps * 32);  // [kRows]
  __shared__ int s_qend;

  const int64_t N = pv.N;
  const int64_t j0 = (int64_t)(blockIdx.x >> 1) * kBlock + (blockIdx.x & 1) * kRows;
  if (j0 >= N) return;
  const int hk = blockIdx.y;
  const int g = hq / hkv;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int idx = tid; idx < kRows * D; idx += kThreads) {
    const int r = idx / D, c = idx % D;
    const int64_t j = j0 + r;
    sK[idx] = j < N ? to_f(k[(j * hkv + hk) * D + c]) : 0.f;
    sV[idx] = j < N ? to_f(v[(j * hkv + hk) * D + c]) : 0.f;
  }
  if (tid == 0) s_qend = 0;
  __syncthreads();
  if (tid < kRows) {
    const int64_t j = j0 + tid;
    const int e = j < N ? pv.E[j] : -1;
    sE[tid] = e;
    atomicMax(&s_qend, e);
  }
  float adk[kPerWarp][NC], adv[kPerWarp][NC];
#pragma unroll
  for (int rr = 0; rr < kPerWarp; ++rr)
#pragma unroll
    for (int cc = 0; cc < NC; ++cc) adk[rr][cc] = adv[rr][cc] = 0.f;
  __syncthreads();
  const int64_t qend = s_qend;
  for (int hh = 0; hh < g; ++hh) {
    const int h = hk * g + hh;
    for (int64_t i0 = j0; i0 < qend; i0 += kChunk) {
      __syncthreads();
      for (int idx = tid; idx < kChunk * D; idx += kThreads) {
        const int ii = idx / D, c = idx % D;
        const int64_t i = i0 + ii;
        const bool in = i < N;
        sQ[ii * DP + c] = in ? to_f(q[(i * hq + h) * D + c]) : 0.f;
        sG[ii * DP + c] = in ? to_f(dout[(i * hq + h) * D + c]) : 0.f;
      }
      if (tid < kChunk) {
        const int64_t i = i0 + tid;
        const bool in = i < N;
        sL[tid] = in ? lse[(int64_t)h * N + i] * kLog2e : 0.f;
        sD[tid] = in ? Dvec[(int64_t)h * N + i] : 0.f;
        sW[tid] = (in && restore) ? (pv.wr ? pv.wr[i] : (float)pv.w[i]) : 1.f;
      }
      __syncthreads();
      const int64_t i = i0 + lane;
#pragma unroll
      for (int rr = 0; rr < kPerWarp; ++rr) {
        const int r = warp * kPerWarp + rr;
        const int64_t j = j0 + r;
        if (j >= N) continue;
        float s = 0.f, dp = 0.f;
#pragma unroll 8
        for (int c = 0; c < D; ++c) {
          s = fmaf(sK[r * D + c], sQ[lane * DP + c], s);
          dp = fmaf(sV[r * D + c], sG[lane * DP + c], dp);
        }
        const bool ok = (i < N) && (j <= i) && (i < (int64_t)sE[r]);
        const float p = ok ? exp2f(s * scale_log2 - sL[lane]) : 0.f;
        const float pw = sW[lane] * p;
        sPW[warp * 32 + lane] = pw;
        sS[warp * 32 + lane] = pw * (dp - sD[lane]);
        __syncwarp();
#pragma unroll
        for (int cc = 0; cc < NC; ++cc) {
          const int c = lane + 32 * cc;
          float a = adv[rr][cc], b = adk[rr][cc];
#pragma unroll 8
          for (int ii = 0; ii < kChunk; ++ii) {
            a = fmaf(sPW[warp * 32 + ii], sG[ii * DP + c], a);
            b = fmaf(sS[warp * 32 + ii], sQ[ii * DP + c], b);
          }
          adv[rr][cc] = a;
          adk[rr][cc] = b;
        }
        __syncwarp();
      }
    }
  }
#pragma unroll
  for (int rr = 0; rr < kPerWarp; ++rr) {
    const int64_t j = j0 + warp * kPerWarp + rr;
    if (j >= N) continue;
#pragma unroll
    for (int cc = 0; cc < NC; ++cc) {
      dk[(j * hkv + hk) * D + lane + 32 * cc] = from_f<T>(adk[rr][cc] * scale);
      dv[(j * hkv + hk) * D + lane + 32 * cc] = from_f<T>(adv[rr][cc]);
    }
  }
}

template <int D> constexpr size_t fwd_smem() { return (size_t)(kRows * D + kChunk * (D + 1) + kChunk * D + kWarps * 32 + kChunk) * 4; }
template <int D> constexpr size_t dq_smem() { return (size_t)(2 * kRows * D + 2 * kChunk * (D + 1) + kWarps * 32 + kChunk) * 4; }
template <int D> constexpr size_t dkdv_smem() {
  return (size_t)(2 * kRows * D + 2 * kChunk * (D + 1) + 3 * kChunk + 2 * kWarps * 32 + kRows) * 4;
}

PackView view(const tt_packed& pk) {
  return PackView{pk.n_tokens, pk.w, pk.wr, pk.E, pk.kblk_maxE, pk.fwd_cnt, pk.fwd_list};
}

template <typename T, int D>
tt_status fwd_impl(const tt_packed& pk, const void* q, const void* k, const void* v, int hq, int hkv, float scale,
                   void* o, float* lse, cudaStream_t st) {
  auto kern = simt_fwd_kernel<T, D>;
  const size_t sm = fwd_smem<D>();
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  dim3 grid(pk.n_blk * 2, hq);
  kern<<<grid, kThreads, sm, st>>>(view(pk), (const T*)q, (const T*)k, (const T*)v, hq, hkv, scale * kLog2e, (T*)o, lse);
  count_launch();
  return check_launch("simt_fwd_kernel");
}

template <typename T, int D>
tt_status bwd_impl(const tt_packed& pk, const void* q, const void* k, const void* v, const float* lse, const float* Dvec,
                   const void* dout, int restore, int hq, int hkv, float scale, void* dq, void* dk, void* dv,
                   cudaStream_t st) {
  auto kq = simt_dq_kernel<T, D>;
  auto kkv = simt_dkdv_kernel<T, D>;
  cudaFuncSetAttribute(kq, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dq_smem<D>());
  cudaFuncSetAttribute(kkv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dkdv_smem<D>());
  kq<<<dim3(pk.n_blk * 2, hq), kThreads, dq_smem<D>(), st>>>(view(pk), (const T*)q, (const T*)k, (const T*)v, lse, Dvec,
                                                            (const T*)dout, restore, hq, hkv, scale, scale * kLog2e, (T*)dq);
  count_launch();
  tt_status s = check_launch("simt_dq_kernel");
  if (s) return s;
  kkv<<<dim3(pk.n_blk * 2, hkv), kThreads, dkdv_smem<D>(), st>>>(view(pk), (const T*)q, (const T*)k, (const T*)v, lse,
                                                                 Dvec, (const T*)dout, restore, hq, hkv, scale,
                                                                 scale * kLog2e, (T*)dk, (T*)dv);
  count_launch();
  return check_launch("simt_dkdv_kernel");
}

}  // namespace

tt_status simt_attn_fwd(const tt_packed& pk, const void* q, const void* k, const void* v, tt_dtype dt, int hq, int hkv,
                        int d, float scale, void* o, float* lse, cudaStream_t st) {
  if (dt == TT_FP32 && d == 128) return fwd_impl<float, 128>(pk, q, k, v, hq, hkv, scale, o, lse, st);
  if (dt == TT_FP32 && d == 64) return fwd_impl<float, 64>(pk, q, k, v, hq, hkv, scale, o, lse, st);
  if (dt == TT_BF16 && d == 64) return fwd_impl<__nv_bfloat16, 64>(pk, q, k, v, hq, hkv, scale, o, lse, st);
  if (dt == TT_BF16 && d == 128) return fwd_impl<__nv_bfloat16, 128>(pk, q, k, v, hq, hkv, scale, o, lse, st);
  set_error("simt_attn_fwd: unsupported d=%d", d);
  return TT_ERR_UNSUPPORTED;
}

tt_status simt_attn_bwd(const tt_packed& pk, const void* q, const void* k, const void* v, const float* lse,
                        const float* Dvec, const void* dout, int restore, tt_dtype dt, int hq, int hkv, int d,
                        float scale, void* dq, void* dk, void* dv, cudaStream_t st) {
  if (dt == TT_FP32 && d == 128)
    return bwd_impl<float, 128>(pk, q, k, v, lse, Dvec, dout, restore, hq, hkv, scale, dq, dk, dv, st);
  if (dt == TT_FP32 && d == 64)
    return bwd_impl<float, 64>(pk, q, k, v, lse, Dvec, dout, restore, hq, hkv, scale, dq, dk, dv, st);
  if (dt == TT_BF16 && d == 64)
    return bwd_impl<__nv_bfloat16, 64>(pk, q, k, v, lse, Dvec, dout, restore, hq, hkv, scale, dq, dk, dv, st);
  if (dt == TT_BF16 && d == 128)
    return bwd_impl<__nv_bfloat16, 128>(pk, q, k, v, lse, Dvec, dout, restore, hq, hkv, scale, dq, dk, dv, st);
  set_error("simt_attn_bwd: unsupported d=%d", d);
  return TT_ERR_UNSUPPORTED;
}

}  // namespace tt
