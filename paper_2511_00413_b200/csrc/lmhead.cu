// lmhead.cu — LM head + Gradient-Restoration cross entropy without materialising [N, V] logits
// (the "gradient scaling step before the backward propagation", applied
// inside the loss as per-prediction weights, readings R6-R8, R17, R20; targets R7 / SURVEY App. D).
//
// Given hidden states H [N, D] and the LM-head weight W [V, D] (bf16), computes the same quantities as
// tt_restore_loss on logits X = H W^T, plus the gradients the LM head passes back:
//   loss_t = sum_k omega_k (lse(x_t) - x_t[y_k])                     (tok_loss, sums[0])
//   G_t    = gamma (Omega_t softmax(x_t) - sum_k omega_k e_{y_k})       (dlogits, never stored whole)
//   dH     = G W,    dW = G^T H
// The vocabulary is processed in chunks of Vc columns, so the largest temporary is [N, Vc]:
//   sweep 1, per chunk c:  X_c = H W_c^T (fp32, cuBLASLt — a plain library GEMM)
//                          lm_lse_chunk_kernel: running (max, sum-exp) per row in the log2 domain and
//                          the weighted target logits falling in the chunk
//   finalize:              lse, per-row loss, Omega, deterministic fp64 sums (fixed order)
//   sweep 2, per chunk c:  X_c = H W_c^T again (identical bits: same GEMM, same inputs)
//                          lm_dlogits_chunk_kernel: G_c = gamma (Omega 2^(x log2e - lse2) - ...) -> bf16
//                          dH_acc += G_c W_c (fp32 accumulate), dW_c = G_c^T H (bf16)   (cuBLASLt)
//   dH = bf16(dH_acc)
// Logits stay fp32 end to end (more accurate than a materialised bf16 [N, V]); G is rounded to bf16
// once, as the operand of the two weight-gradient GEMMs.  FLOPs: 4 x 2 N V D (two logits GEMMs, dH,
// dW); HBM for the CE parts ~ N V (4 + 4 + 4 + 2) bytes per pass pair, small next to the GEMMs.
#include <cublasLt.h>

#include <algorithm>
#include <cmath>
#include <mutex>
#include <unordered_map>

#include "tt_internal.cuh"

namespace tt {
namespace {

constexpr int kLmThreads = 256;

struct LmRow {  // per-row state across chunks (log2 domain)
  float m, s, tx, pad;
};

struct LmArgs {
  int64_t N;
  int V, c0, nc, ld;  // chunk columns [c0, c0 + nc), row stride ld (>= nc, multiple of 4)
  const int32_t* tok;
  const uint8_t* node_mask;
  int boundary_mode;
  float gamma;
  const int32_t* w;
  const float* wr;
  const int32_t *node, *node_start, *node_len, *succ_ptr, *succ_tok;
};

// the k-th target (packed index) of row t, or -1 if masked; nt = number of candidate targets
__device__ __forceinline__ int lm_ntargets(const LmArgs& a, int64_t t, bool& last, int& sb) {
  const int32_t u = a.node[t];
  last = t == (int64_t)a.node_start[u] + a.node_len[u] - 1;
  if (!last) return 1;
  sb = a.succ_ptr[u];
  const int se = a.succ_ptr[u + 1];
  if (a.boundary_mode == 1) {  // exclude when the trajectories continue to more than one next token
    int live = 0;
    for (int k = sb; k < se && live < 2; ++k) live += (a.w[a.succ_tok[k]] > 0);
    if (live > 1) return 0;
  }
  return se - sb;
}
__device__ __forceinline__ int lm_target(const LmArgs& a, int64_t t, bool last, int sb, int k) {
  const int tg = last ? a.succ_tok[sb + k] : (int)(t + 1);
  if (a.node_mask && !a.node_mask[a.node[tg]]) return -1;
  return tg;
}
__device__ __forceinline__ float lm_omega(const LmArgs& a, int tg) { return a.wr ? a.wr[tg] : (float)a.w[tg]; }

__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// block-wide reductions (kLmThreads threads); every thread gets the result
template <bool kMax>
__device__ __forceinline__ float block_reduce(float v, float* sh) {
  for (int o = 16; o > 0; o >>= 1) {
    const float u = __shfl_xor_sync(0xffffffffu, v, o);
    v = kMax ? fmaxf(v, u) : v + u;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < kLmThreads / 32 ? sh[lane] : (kMax ? -INFINITY : 0.f);
    for (int o = 16; o > 0; o >>= 1) {
      const float u = __shfl_xor_sync(0xffffffffu, v, o);
      v = kMax ? fmaxf(v, u) : v + u;
    }
    if (lane == 0) sh[0] = v;
  }
  __syncthreads();
  v = sh[0];
  __syncthreads();
  return v;
}

// sweep 1: one CTA per row; chunk max / sum-exp merged into the row state, weighted target logits
__global__ void __launch_bounds__(kLmThreads) lm_lse_chunk_kernel(const LmArgs a, const float* __restrict__ X,
                                                                  LmRow* __restrict__ st, int first) {
  __shared__ float sh[32];
  const int64_t t = blockIdx.x;
  const float* x = X + t * (int64_t)a.ld;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  const int n4 = a.nc / 4;
  float m = -INFINITY;
  for (int v = threadIdx.x; v < n4; v += kLmThreads) {
    const float4 q = x4[v];
    m = fmaxf(m, fmaxf(fmaxf(q.x, q.y), fmaxf(q.z, q.w)));
  }
  for (int c = 4 * n4 + threadIdx.x; c < a.nc; c += kLmThreads) m = fmaxf(m, x[c]);
  m = block_reduce<true>(m, sh) * kLog2e;
  float s = 0.f;
  for (int v = threadIdx.x; v < n4; v += kLmThreads) {
    const float4 q = x4[v];
    s += ex2f(fmaf(q.x, kLog2e, -m)) + ex2f(fmaf(q.y, kLog2e, -m)) + ex2f(fmaf(q.z, kLog2e, -m)) +
         ex2f(fmaf(q.w, kLog2e, -m));
  }
  for (int c = 4 * n4 + threadIdx.x; c < a.nc; c += kLmThreads) s += ex2f(fmaf(x[c], kLog2e, -m));
  s = block_reduce<false>(s, sh);
  // weighted target logits in this chunk
  bool last = false;
  int sb = 0;
  const int nt = lm_ntargets(a, t, last, sb);
  float tx = 0.f;
  for (int k = threadIdx.x; k < nt; k += kLmThreads) {
    const int tg = lm_target(a, t, last, sb, k);
    if (tg < 0) continue;
    const int y = a.tok[tg];
    if (y >= a.c0 && y < a.c0 + a.nc) tx += lm_omega(a, tg) * x[y - a.c0];
  }
  tx = block_reduce<false>(tx, sh);
  if (threadIdx.x == 0) {
    LmRow r = first ? LmRow{-INFINITY, 0.f, 0.f, 0.f} : st[t];
    const float mm = fmaxf(r.m, m);
    r.s = (mm == -INFINITY) ? 0.f : r.s * ex2f(r.m - mm) + s * ex2f(m - mm);
    r.m = mm;
    r.tx += tx;
    st[t] = r;
  }
}

// per row: Omega, lse (log2 domain, kept in st[t].m), loss row, error flag
__global__ void __launch_bounds__(kLmThreads) lm_finalize_kernel(const LmArgs a, LmRow* __restrict__ st,
                                                                 float* __restrict__ omega_row, float* __restrict__ ws_loss,
                                                                 float* __restrict__ ws_omega, float* __restrict__ tok_loss,
                                                                 int32_t* d_err) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= a.N) return;
  bool last = false;
  int sb = 0;
  const int nt = lm_ntargets(a, t, last, sb);
  float om = 0.f;
  bool bad = false;
  for (int k = 0; k < nt; ++k) {
    const int tg = lm_target(a, t, last, sb, k);
    if (tg < 0) continue;
    const int y = a.tok[tg];
    bad |= (y < 0 || y >= a.V);
    om += lm_omega(a, tg);
  }
  LmRow r = st[t];
  const float lse2 = r.m + log2f(r.s);
  const float lv = bad ? __int_as_float(0x7fc00000) : (om == 0.f ? 0.f : om * lse2 * kLn2 - r.tx);
  if (bad && d_err) atomicExch(d_err, 1);
  ws_loss[t] = lv;
  ws_omega[t] = bad ? 0.f : om;
  if (tok_loss) tok_loss[t] = lv;
  omega_row[t] = bad ? 0.f : om;
  r.m = lse2;  // sweep 2 reads lse2 from here
  st[t] = r;
}

// sweep 2: G_c = gamma (Omega 2^(x log2e - lse2) - sum_{k: y_k = col} omega_k) -> bf16 [N, ldo]
__global__ void __launch_bounds__(kLmThreads) lm_dlogits_chunk_kernel(const LmArgs a, const float* __restrict__ X,
                                                                      const LmRow* __restrict__ st,
                                                                      const float* __restrict__ omega_row,
                                                                      __nv_bfloat16* __restrict__ G, int ldo) {
  const int64_t t = blockIdx.x;
  const float* x = X + t * (int64_t)a.ld;
  __nv_bfloat16* g = G + t * (int64_t)ldo;
  const float lse2 = st[t].m;
  const float gO = a.gamma * omega_row[t];
  const int n2 = a.nc / 2;
  for (int v = threadIdx.x; v < n2; v += kLmThreads) {
    const float2 q = reinterpret_cast<const float2*>(x)[v];
    reinterpret_cast<__nv_bfloat162*>(g)[v] =
        __floats2bfloat162_rn(gO * ex2f(fmaf(q.x, kLog2e, -lse2)), gO * ex2f(fmaf(q.y, kLog2e, -lse2)));
  }
  if ((a.nc & 1) && threadIdx.x == 0) g[a.nc - 1] = __float2bfloat16_rn(gO * ex2f(fmaf(x[a.nc - 1], kLog2e, -lse2)));
  for (int c = a.nc + threadIdx.x; c < ldo; c += kLmThreads) g[c] = __float2bfloat16_rn(0.f);  // padding columns
  __syncthreads();
  if (gO == 0.f && omega_row[t] == 0.f) return;  // no prediction (or a bad target): row is all zeros
  bool last = false;
  int sb = 0;
  const int nt = lm_ntargets(a, t, last, sb);
  for (int k = threadIdx.x; k < nt; k += kLmThreads) {
    const int tg = lm_target(a, t, last, sb, k);
    if (tg < 0) continue;
    const int y = a.tok[tg];
    if (y < a.c0 || y >= a.c0 + a.nc) continue;
    // first occurrence of y among the row's targets writes the combined value
    bool first = true;
    float om_y = 0.f;
    for (int k2 = 0; k2 < nt; ++k2) {
      const int tg2 = lm_target(a, t, last, sb, k2);
      if (tg2 < 0 || a.tok[tg2] != y) continue;
      if (k2 < k) first = false;
      om_y += lm_omega(a, tg2);
    }
    if (first) {
      const float py = ex2f(fmaf(x[y - a.c0], kLog2e, -lse2));
      g[y - a.c0] = __float2bfloat16_rn(a.gamma * (omega_row[t] * py - om_y));
    }
  }
}

__global__ void __launch_bounds__(256) lm_convert_kernel(const float4* __restrict__ in, uint2* __restrict__ out,
                                                         int64_t n4) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = in[i];
    __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
    out[i] = make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
  }
}

// ---------------------------------------------------------------------------- cuBLASLt GEMMs
// One cuBLASLt handle per (thread, device), created on first use (the library's only cached
// state besides the thread-local error string).
cublasLtHandle_t lt_handle() {
  thread_local std::unordered_map<int, cublasLtHandle_t> handles;
  int dev = 0;
  cudaGetDevice(&dev);
  auto it = handles.find(dev);
  if (it != handles.end()) return it->second;
  cublasLtHandle_t h = nullptr;
  if (cublasLtCreate(&h) != CUBLAS_STATUS_SUCCESS) return nullptr;
  handles[dev] = h;
  return h;
}

// column-major D[m x n] = alpha op(A) op(B) + beta D; A/B bf16, D fp32 or bf16, fp32 compute.
// lda/ldb/ldd are the leading dimensions of the STORED matrices.
tt_status lt_gemm(bool ta, bool tb, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda, const void* B,
                  int64_t ldb, void* D, int64_t ldd, cudaDataType_t dtype, float beta, void* ws, size_t wsz,
                  cudaStream_t st) {
  cublasLtHandle_t h = lt_handle();
  if (!h) { set_error("cublasLtCreate failed"); return TT_ERR_CUDA; }
  cublasLtMatmulDesc_t op = nullptr;
  cublasLtMatrixLayout_t la = nullptr, lb = nullptr, ld = nullptr;
  cublasLtMatmulPreference_t pref = nullptr;
  tt_status s = TT_OK;
  const cublasOperation_t opa = ta ? CUBLAS_OP_T : CUBLAS_OP_N, opb = tb ? CUBLAS_OP_T : CUBLAS_OP_N;
  const float alpha = 1.f;
  cublasLtMatmulHeuristicResult_t res = {};
  int nres = 0;
  cublasStatus_t e = cublasLtMatmulDescCreate(&op, CUBLAS_COMPUTE_32F, CUDA_R_32F);
  if (e == CUBLAS_STATUS_SUCCESS) e = cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSA, &opa, sizeof(opa));
  if (e == CUBLAS_STATUS_SUCCESS) e = cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSB, &opb, sizeof(opb));
  if (e == CUBLAS_STATUS_SUCCESS) e = cublasLtMatrixLayoutCreate(&la, CUDA_R_16BF, ta ? k : m, ta ? m : k, lda);
  if (e == CUBLAS_STATUS_SUCCESS) e = cublasLtMatrixLayoutCreate(&lb, CUDA_R_16BF, tb ? n : k, tb ? k : n, ldb);
  if (e == CUBLAS_STATUS_SUCCESS) e = cublasLtMatrixLayoutCreate(&ld, dtype, m, n, ldd);
  if (e == CUBLAS_STATUS_SUCCESS) e = cublasLtMatmulPreferenceCreate(&pref);
  if (e == CUBLAS_STATUS_SUCCESS)
    e = cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &wsz, sizeof(wsz));
  if (e == CUBLAS_STATUS_SUCCESS) e = cublasLtMatmulAlgoGetHeuristic(h, op, la, lb, ld, ld, pref, 1, &res, &nres);
  if (e == CUBLAS_STATUS_SUCCESS && nres == 0) e = CUBLAS_STATUS_NOT_SUPPORTED;
  if (e == CUBLAS_STATUS_SUCCESS)
    e = cublasLtMatmul(h, op, &alpha, A, la, B, lb, &beta, D, ld, D, ld, &res.algo, ws, wsz, st);
  if (e != CUBLAS_STATUS_SUCCESS) {
    set_error("cuBLASLt matmul (m=%lld n=%lld k=%lld) failed: status %d", (long long)m, (long long)n, (long long)k, (int)e);
    s = TT_ERR_CUDA;
  }
  if (pref) cublasLtMatmulPreferenceDestroy(pref);
  if (ld) cublasLtMatrixLayoutDestroy(ld);
  if (lb) cublasLtMatrixLayoutDestroy(lb);
  if (la) cublasLtMatrixLayoutDestroy(la);
  if (op) cublasLtMatmulDescDestroy(op);
  return s;
}

inline size_t al256(size_t x) { return (x + 255) & ~size_t(255); }
constexpr size_t kLtWorkspace = 32u << 20;

struct LmLayout {
  size_t X, G, dh, st, om, wl, wo, lt, total;
};
LmLayout lm_layout(int64_t N, int D, int Vc) {
  const int ldc = (Vc + 7) / 8 * 8;
  LmLayout L;
  size_t o = 0;
  L.X = o;  o += al256((size_t)N * ldc * 4);
  L.G = o;  o += al256((size_t)N * ldc * 2);
  L.dh = o; o += al256((size_t)N * D * 4);
  L.st = o; o += al256((size_t)N * sizeof(LmRow));
  L.om = o; o += al256((size_t)N * 4);
  L.wl = o; o += al256((size_t)N * 4);
  L.wo = o; o += al256((size_t)N * 4);
  L.lt = o; o += kLtWorkspace;
  L.total = o;
  return L;
}

}  // namespace

size_t lmhead_ws_bytes(int64_t N, int D, int V, int Vc) { return lm_layout(N, D, std::min(V, Vc)).total; }

tt_status launch_lmhead_loss(const tt_packed& pk, const __nv_bfloat16* H, const __nv_bfloat16* W, int D, int V, int Vc,
                             const int32_t* tok, const uint8_t* node_mask, int boundary_mode, float gamma,
                             __nv_bfloat16* dH, __nv_bfloat16* dW, float* tok_loss, double* sums, int32_t* d_err,
                             void* ws, cudaStream_t st) {
  const int64_t N = pk.n_tokens;
  Vc = std::min(V, Vc);
  const LmLayout L = lm_layout(N, D, Vc);
  char* w8 = static_cast<char*>(ws);
  float* X = reinterpret_cast<float*>(w8 + L.X);
  __nv_bfloat16* G = reinterpret_cast<__nv_bfloat16*>(w8 + L.G);
  float* dh_acc = reinterpret_cast<float*>(w8 + L.dh);
  LmRow* rs = reinterpret_cast<LmRow*>(w8 + L.st);
  float* om = reinterpret_cast<float*>(w8 + L.om);
  float* ws_loss = reinterpret_cast<float*>(w8 + L.wl);
  float* ws_omega = reinterpret_cast<float*>(w8 + L.wo);
  void* lt_ws = w8 + L.lt;
  LmArgs a{N, V, 0, 0, 0, tok, node_mask, boundary_mode, gamma, pk.w, pk.wr,
           pk.node, pk.node_start, pk.node_len, pk.succ_ptr, pk.succ_tok};
  tt_status s;
  // ---- sweep 1: X_c = H W_c^T (column-major: X_c^T [nc x N] = W_c [nc x D] . H^T), row state ----
  for (int c0 = 0; c0 < V; c0 += Vc) {
    const int nc = std::min(Vc, V - c0), ldc = (nc + 7) / 8 * 8;
    if ((s = lt_gemm(true, false, nc, N, D, W + (int64_t)c0 * D, D, H, D, X, ldc, CUDA_R_32F, 0.f, lt_ws,
                     kLtWorkspace, st)))
      return s;
    a.c0 = c0; a.nc = nc; a.ld = ldc;
    lm_lse_chunk_kernel<<<(unsigned)N, kLmThreads, 0, st>>>(a, X, rs, c0 == 0);
    count_launch();
    if ((s = check_launch("lm_lse_chunk_kernel"))) return s;
  }
  lm_finalize_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(a, rs, om, ws_loss, ws_omega, tok_loss, d_err);
  count_launch();
  if ((s = check_launch("lm_finalize_kernel"))) return s;
  if ((s = launch_loss_sums(N, ws_loss, ws_omega, sums, st))) return s;
  // ---- sweep 2: recompute X_c, G_c, dH_acc += G_c W_c, dW_c = G_c^T H ----
  for (int c0 = 0; c0 < V; c0 += Vc) {
    const int nc = std::min(Vc, V - c0), ldc = (nc + 7) / 8 * 8;
    if ((s = lt_gemm(true, false, nc, N, D, W + (int64_t)c0 * D, D, H, D, X, ldc, CUDA_R_32F, 0.f, lt_ws,
                     kLtWorkspace, st)))
      return s;
    a.c0 = c0; a.nc = nc; a.ld = ldc;
    lm_dlogits_chunk_kernel<<<(unsigned)N, kLmThreads, 0, st>>>(a, X, rs, om, G, ldc);
    count_launch();
    if ((s = check_launch("lm_dlogits_chunk_kernel"))) return s;
    // dH^T [D x N] (+)= W_c^T [D x nc] . G_c^T [nc x N]
    if ((s = lt_gemm(false, false, D, N, nc, W + (int64_t)c0 * D, D, G, ldc, dh_acc, D, CUDA_R_32F, c0 == 0 ? 0.f : 1.f,
                     lt_ws, kLtWorkspace, st)))
      return s;
    // dW_c^T [D x nc] = H^T [D x N] . G_c [N x nc]
    if ((s = lt_gemm(false, true, D, nc, N, H, D, G, ldc, dW + (int64_t)c0 * D, D, CUDA_R_16BF, 0.f, lt_ws,
                     kLtWorkspace, st)))
      return s;
  }
  const int64_t n4 = N * (int64_t)D / 4;
  lm_convert_kernel<<<(unsigned)std::min<int64_t>((n4 + 255) / 256, 148 * 16), 256, 0, st>>>(
      reinterpret_cast<const float4*>(dh_acc), reinterpret_cast<uint2*>(dH), n4);
  count_launch();
  return check_launch("lm_convert_kernel");
}

}  // namespace tt
