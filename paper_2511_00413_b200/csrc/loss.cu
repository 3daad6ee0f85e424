// loss.cu — Gradient-Restoration loss: weighted next-token cross entropy
// and its gradient, HBM-bound, one persistent CTA per row stream.
//
// The paper restores gradients by "insert[ing] a gradient scaling step before the backward
// propagation" that multiplies each node's gradient by its reuse count.  At the
// loss (R6) this is exactly a per-prediction weight omega_k = w[target]: every one
// of the w[target] trajectories through the predicting token t continues to that target, so
//   loss_t    = sum_k omega_k (lse(x_t) - x_t[y_k])
//   dlogits_t = gamma (Omega_t softmax(x_t) - sum_k omega_k e_{y_k})
// Targets (R7): t+1 inside a node; at a node's last token every continuation (succ list).
//
// Memory plan per row (V = 151,936 bf16 = 297 KB):  pass 1 streams the row from HBM with 32-byte
// vector loads marked L2::evict_last (online max / sum-exp in the log2 domain, one max pass and
// at most one rescale per vector); pass 2 re-reads it from L2 (one 1024-thread CTA per SM keeps
// 148 rows = 44 MB in flight, well under the 126 MB L2) marked evict_first, and writes dlogits
// (evict_first; may alias logits).  HBM
// traffic is therefore ~4 V bytes / row.  Rows with no target (Omega_t = 0, e.g.
// the last token of every trajectory) skip both reads and only write zeros.
#include <algorithm>
#include <cstdio>
#include <unordered_map>
#include <utility>
#include <cstdlib>

#include <cuda_fp16.h>

#include "tt_internal.cuh"
#include "sm100_ptx.cuh"

namespace tt {
namespace {

constexpr int kLossThreads = 1024;
constexpr int kMaxTargets = 1024;

// W bf16 logits per thread-vector: 16 (32-byte .v8.b32 accesses; needs 32-byte aligned rows) or 8.
template <int W> struct Vec { uint32_t u[W / 2]; };

// pass 1: streaming read that asks L2 to keep the line (it is re-read by pass 2)
// boundary_mode 1 excludes a node's last token when the trajectories through it continue
// to more than one next token: continuations are counted only if some trajectory passes through them
// (w > 0: a child subtree with no trajectory end is no branch), matching the per-branch definition
__device__ __forceinline__ bool diverges(const int32_t* succ_tok, int b, int e, const int32_t* w) {
  int live = 0;
  for (int k = b; k < e && live < 2; ++k) live += (w[succ_tok[k]] > 0);
  return live > 1;
}

template <int W> __device__ __forceinline__ Vec<W> ld_keep(const __nv_bfloat16* p) {
  Vec<W> r;
  if constexpr (W == 16)
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_last.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r.u[0]), "=r"(r.u[1]), "=r"(r.u[2]), "=r"(r.u[3]), "=r"(r.u[4]), "=r"(r.u[5]), "=r"(r.u[6]),
                   "=r"(r.u[7])
                 : "l"(p));
  else
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.u[0]), "=r"(r.u[1]), "=r"(r.u[2]), "=r"(r.u[3])
                 : "l"(p));
  return r;
}
// pass 2: coherent read (dlogits may alias logits: each thread reads, then overwrites, its own
// vectors), last use of the line
template <int W> __device__ __forceinline__ Vec<W> ld_last(const __nv_bfloat16* p) {
  Vec<W> r;
  if constexpr (W == 16)
    asm volatile("ld.global.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r.u[0]), "=r"(r.u[1]), "=r"(r.u[2]), "=r"(r.u[3]), "=r"(r.u[4]), "=r"(r.u[5]), "=r"(r.u[6]),
                   "=r"(r.u[7])
                 : "l"(p)
                 : "memory");
  else
    asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.u[0]), "=r"(r.u[1]), "=r"(r.u[2]), "=r"(r.u[3])
                 : "l"(p)
                 : "memory");
  return r;
}
template <int W> __device__ __forceinline__ void st_vec(__nv_bfloat16* p, const Vec<W>& r) {
  if constexpr (W == 16)
    asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(r.u[0]), "r"(r.u[1]),
                 "r"(r.u[2]), "r"(r.u[3]), "r"(r.u[4]), "r"(r.u[5]), "r"(r.u[6]), "r"(r.u[7])
                 : "memory");
  else
    asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(r.u[0]), "r"(r.u[1]),
                 "r"(r.u[2]), "r"(r.u[3])
                 : "memory");
}
__device__ __forceinline__ float2 bf2f(uint32_t u) {
  return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u));
}
__device__ __forceinline__ uint32_t f2bf(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ uint32_t f2h(float lo, float hi) {
  __half2 v = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// (m, s) <- (m, s) (+) one vector of logits, log2 domain: one max pass, at most one rescale
// KP1: pairs (of W/2) whose exponentials run on the FMA pipe (degree-3 polynomial, max rel. error
// 7.5e-5 per term; with 1 of 4 pairs the sum-exp, hence the lse, moves by <= 1.9e-5 relative)
template <int W, int KP1 = 0> __device__ __forceinline__ void accum(float& m, float& s, const Vec<W>& r) {
  float x[W];
#pragma unroll
  for (int t = 0; t < W / 2; ++t) {
    const float2 f = bf2f(r.u[t]);
    x[2 * t] = f.x * kLog2e;
    x[2 * t + 1] = f.y * kLog2e;
  }
  float cm = x[0];
#pragma unroll
  for (int t = 1; t < W; ++t) cm = fmaxf(cm, x[t]);
  if (cm > m) {
    s *= ex2f(m - cm);  // m = -inf -> 0
    m = cm;
  }
  float a = 0.f, b = 0.f;
#pragma unroll
  for (int t = 0; t < W; t += 2) {
    if (t / 2 >= W / 2 - KP1) {
      const float2 e = sm100::exp2_poly2(make_float2(x[t] - m, x[t + 1] - m));
      a += e.x;
      b += e.y;
    } else {
      a += ex2f(x[t] - m);
      b += ex2f(x[t + 1] - m);
    }
  }
  s += a + b;
}

template <int W>
__global__ void __launch_bounds__(kLossThreads) loss_kernel(
    int64_t N, const __nv_bfloat16* logits, int64_t ld, int V, const int32_t* __restrict__ tok,
    const uint8_t* __restrict__ node_mask, int boundary_mode, float gamma, const int32_t* __restrict__ w, const float* __restrict__ wr,
    const int32_t* __restrict__ node, const int32_t* __restrict__ node_start, const int32_t* __restrict__ node_len,
    const int32_t* __restrict__ succ_ptr, const int32_t* __restrict__ succ_tok, __nv_bfloat16* dlogits,
    float* __restrict__ tok_loss, float* __restrict__ ws_loss, float* __restrict__ ws_omega, int32_t* d_err) {
  __shared__ int s_y[kMaxTargets];
  __shared__ float s_om[kMaxTargets];
  __shared__ float s_xy[kMaxTargets];
  __shared__ int s_nt;
  __shared__ float s_red[2][kLossThreads / 32];
  __shared__ float s_lse;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int VW = V - V % W;  // vectorised prefix
  constexpr int STEP = kLossThreads * W;

  for (int64_t row = blockIdx.x; row < N; row += gridDim.x) {
    // ---- targets of this row (R7, R17, boundary mode) ----
    if (tid == 0) {
      const int32_t u = node[row];
      const bool last = row == (int64_t)node_start[u] + node_len[u] - 1;
      int nt = 0;
      if (!last) {
        const int64_t tg = row + 1;
        if (!node_mask || node_mask[node[tg]]) { s_y[0] = (int)tg; nt = 1; }
      } else {
        const int b = succ_ptr[u], e = succ_ptr[u + 1];
        if (!(boundary_mode == 1 && diverges(succ_tok, b, e, w))) {
          for (int k = b; k < e; ++k) {
            const int tg = succ_tok[k];
            if (!node_mask || node_mask[node[tg]]) s_y[nt++] = tg;
          }
        }
      }
      s_nt = nt;
    }
    __syncthreads();
    const int nt = s_nt;
    // packed target index -> (token id, weight = tree-scale of the target)
    float om_part = 0.f;
    bool bad = false;
    for (int k = tid; k < nt; k += kLossThreads) {
      const int tg = s_y[k];
      const int y = tok[tg];
      const float om = wr ? wr[tg] : (float)w[tg];
      bad |= (y < 0 || y >= V);
      s_y[k] = y;
      s_om[k] = om;
      om_part += om;
    }
    const __nv_bfloat16* x = logits + row * ld;
    __nv_bfloat16* dx = dlogits + row * ld;
    for (int o = 16; o > 0; o >>= 1) om_part += __shfl_xor_sync(0xffffffffu, om_part, o);
    const int bad_any = __syncthreads_or(bad);
    if (lane == 0) s_red[0][warp] = om_part;
    __syncthreads();
    float Omega = 0.f;
    for (int k = 0; k < kLossThreads / 32; ++k) Omega += s_red[0][k];
    __syncthreads();  // s_red is reused below
    if (Omega == 0.f || bad_any) {
      // no prediction from this row (or an invalid target id): zero gradient, no logits read
      Vec<W> z;
#pragma unroll
      for (int t = 0; t < W / 2; ++t) z.u[t] = 0u;
      for (int c = tid * W; c < VW; c += STEP) st_vec<W>(dx + c, z);
      for (int c = VW + tid; c < V; c += kLossThreads) dx[c] = __float2bfloat16_rn(0.f);
      if (tid == 0) {
        const float lv = bad_any ? __int_as_float(0x7fc00000) : 0.f;
        if (bad_any && d_err) atomicExch(d_err, 1);
        ws_loss[row] = lv;
        ws_omega[row] = bad_any ? 0.f : Omega;
        if (tok_loss) tok_loss[row] = lv;
      }
      __syncthreads();
      continue;
    }
    // ---- pass 1: online max / sum-exp, two vectors in flight per thread ----
    float m = -INFINITY, sum = 0.f;
    int c = tid * W;
    for (; c + STEP < VW; c += 2 * STEP) {
      const Vec<W> a = ld_keep<W>(x + c), b = ld_keep<W>(x + c + STEP);
      accum<W>(m, sum, a);
      accum<W>(m, sum, b);
    }
    for (; c < VW; c += STEP) accum<W>(m, sum, ld_keep<W>(x + c));
    for (int cc = VW + tid; cc < V; cc += kLossThreads) {
      const float x2 = __bfloat162float(x[cc]) * kLog2e;
      if (x2 > m) { sum = sum * ex2f(m - x2) + 1.f; m = x2; } else { sum += ex2f(x2 - m); }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
      const float s2 = __shfl_xor_sync(0xffffffffu, sum, o);
      const float mm = fmaxf(m, m2);
      sum = (mm == -INFINITY) ? 0.f : sum * ex2f(m - mm) + s2 * ex2f(m2 - mm);
      m = mm;
    }
    if (lane == 0) { s_red[0][warp] = m; s_red[1][warp] = sum; }
    __syncthreads();
    if (tid == 0) {
      float M = -INFINITY, S = 0.f;
      for (int k = 0; k < kLossThreads / 32; ++k) {
        const float m2 = s_red[0][k], s2 = s_red[1][k];
        const float mm = fmaxf(M, m2);
        S = (mm == -INFINITY) ? 0.f : S * ex2f(M - mm) + s2 * ex2f(m2 - mm);
        M = mm;
      }
      s_lse = M + log2f(S);  // log2 units
    }
    __syncthreads();
    const float lse2 = s_lse;
    // ---- loss: read the target logits before pass 2 may overwrite them (aliasing) ----
    float lpart = 0.f;
    for (int k = tid; k < nt; k += kLossThreads) {
      const float xy = __bfloat162float(x[s_y[k]]);
      s_xy[k] = xy;
      lpart += s_om[k] * (lse2 * kLn2 - xy);
    }
    for (int o = 16; o > 0; o >>= 1) lpart += __shfl_xor_sync(0xffffffffu, lpart, o);
    __syncthreads();
    if (lane == 0) s_red[1][warp] = lpart;
    __syncthreads();
    // ---- pass 2: dlogits = gamma * Omega * softmax (target entries fixed up below) ----
    const float gO = gamma * Omega;
    for (c = tid * W; c < VW; c += STEP) {
      const Vec<W> a = ld_last<W>(x + c);
      Vec<W> o;
#pragma unroll
      for (int t = 0; t < W / 2; ++t) {
        const float2 f = bf2f(a.u[t]);
        o.u[t] = f2bf(gO * ex2f(fmaf(f.x, kLog2e, -lse2)), gO * ex2f(fmaf(f.y, kLog2e, -lse2)));
      }
      st_vec<W>(dx + c, o);
    }
    for (int cc = VW + tid; cc < V; cc += kLossThreads)
      dx[cc] = __float2bfloat16_rn(gO * ex2f(fmaf(__bfloat162float(x[cc]), kLog2e, -lse2)));
    __syncthreads();
    // ---- fix-up: dlogits[y] = gamma (Omega p_y - sum_{k: y_k = y} omega_k), once per distinct y ----
    for (int k = tid; k < nt; k += kLossThreads) {
      const int y = s_y[k];
      bool first = true;
      float om_y = 0.f;
      for (int k2 = 0; k2 < nt; ++k2) {
        if (s_y[k2] == y) {
          if (k2 < k) first = false;
          om_y += s_om[k2];
        }
      }
      if (first) {
        const float py = ex2f(fmaf(s_xy[k], kLog2e, -lse2));
        dx[y] = __float2bfloat16_rn(gamma * (Omega * py - om_y));
      }
    }
    if (tid == 0) {
      float L = 0.f;
      for (int k = 0; k < kLossThreads / 32; ++k) L += s_red[1][k];
      ws_loss[row] = L;
      ws_omega[row] = Omega;
      if (tok_loss) tok_loss[row] = L;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------------------------
// Pipelined variant (V % 16 == 0, 32-byte aligned rows): a producer warp streams every row in 32 KB
// chunks into a 4-slot shared-memory ring with TMA bulk copies (L2 evict_last policy, so pass 2 finds
// the row in L2); a meta warp resolves the targets and weights of the upcoming rows into a 2-slot
// metadata ring; 16 compute warps run pass 1 out of shared memory (picking up the target logits on
// the way), then pass 2 re-reads the row from L2 and writes dlogits while the producer is already
// prefetching the next row.
// ---------------------------------------------------------------------------------------------
constexpr int kPipeCompute = 512;                 // compute threads
constexpr int kPipeThreads = kPipeCompute + 64;   // + producer warp + meta warp
constexpr int kChunkElems = 16384;                // 32 KB of bf16
constexpr int kRing = 4;
constexpr int kMetaSlots = 2;                     // rows of metadata the meta warp runs ahead
constexpr size_t kPipeSmem = (size_t)kRing * kChunkElems * 2 + (2 * kRing + 2 * kMetaSlots) * 8;

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init_(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_wait_(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                   smem_addr(b)),
               "r"(ph)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(bytes) : "memory");
}

__global__ void __launch_bounds__(kPipeThreads, 1) loss_pipe_kernel(
    int64_t N, const __nv_bfloat16* logits, int64_t ld, int V, const int32_t* __restrict__ tok,
    const uint8_t* __restrict__ node_mask, int boundary_mode, float gamma, const int32_t* __restrict__ w, const float* __restrict__ wr,
    const int32_t* __restrict__ node, const int32_t* __restrict__ node_start, const int32_t* __restrict__ node_len,
    const int32_t* __restrict__ succ_ptr, const int32_t* __restrict__ succ_tok, __nv_bfloat16* dlogits,
    float* __restrict__ tok_loss, float* __restrict__ ws_loss, float* __restrict__ ws_omega, int32_t* d_err,
    int64_t row_begin) {
  extern __shared__ __align__(128) uint8_t lsm[];
  __nv_bfloat16* ring = reinterpret_cast<__nv_bfloat16*>(lsm);            // kRing x 32 KB
  uint64_t* full = reinterpret_cast<uint64_t*>(lsm + kRing * kChunkElems * 2);
  uint64_t* empty = full + kRing;
  uint64_t* mfull = empty + kRing;    // [kMetaSlots] row metadata ready
  uint64_t* mfree = mfull + kMetaSlots;  // [kMetaSlots] row metadata consumed
  __shared__ int s_y[kMetaSlots][kMaxTargets];     // target token ids (the meta warp resolves tok[])
  __shared__ float s_om[kMetaSlots][kMaxTargets];  // target weights omega_k
  __shared__ float s_xy[kMaxTargets];              // target logits (read from the ring in pass 1)
  __shared__ int s_hdr[kMetaSlots][2];             // nt, bad
  __shared__ float s_Om[kMetaSlots];               // Omega
  __shared__ float s_red[2][kPipeCompute / 32];
  __shared__ float s_lse;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nchunk = (V + kChunkElems - 1) / kChunkElems;
  if (tid == 0) {
    for (int k = 0; k < kRing; ++k) { mbar_init_(&full[k], 1); mbar_init_(&empty[k], kPipeCompute); }
    for (int k = 0; k < kMetaSlots; ++k) { mbar_init_(&mfull[k], 32); mbar_init_(&mfree[k], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kPipeCompute / 32) {
    // ============ producer warp: stream every row of this CTA, chunk by chunk ============
    if (lane == 0) {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
      int g = 0;  // global chunk counter (ring slot = g % kRing)
      for (int64_t row = row_begin + blockIdx.x; row < N; row += gridDim.x) {
        const __nv_bfloat16* x = logits + row * ld;
        for (int c = 0; c < nchunk; ++c, ++g) {
          const int slot = g % kRing;
          if (g >= kRing) mbar_wait_(&empty[slot], ((g / kRing) - 1) & 1);
          const int n = min(kChunkElems, V - c * kChunkElems);
          mbar_expect_(&full[slot], (uint32_t)n * 2);
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
                  smem_addr(ring + slot * kChunkElems)),
              "l"(x + (int64_t)c * kChunkElems), "r"(n * 2), "r"(smem_addr(&full[slot])), "l"(pol)
              : "memory");
        }
      }
    }
    return;
  }
  if (warp == kPipeCompute / 32 + 1) {
    // ============ meta warp: targets / weights of the upcoming rows (R7, R17, boundary), a row ahead
    //              of the compute warps so its chain of dependent global loads is off their path ====
    int it = 0;
    for (int64_t row = row_begin + blockIdx.x; row < N; row += gridDim.x, ++it) {
      const int sl = it % kMetaSlots;
      if (it >= kMetaSlots) mbar_wait_(&mfree[sl], (uint32_t)(((it / kMetaSlots) - 1) & 1));
      int nt = 0;
      if (lane == 0) {
        const int32_t u = node[row];
        const bool last = row == (int64_t)node_start[u] + node_len[u] - 1;
        if (!last) {
          const int64_t tg = row + 1;
          if (!node_mask || node_mask[node[tg]]) { s_y[sl][0] = (int)tg; nt = 1; }
        } else {
          const int b = succ_ptr[u], e = succ_ptr[u + 1];
          if (!(boundary_mode == 1 && diverges(succ_tok, b, e, w))) {
            for (int k = b; k < e; ++k) {
              const int tg = succ_tok[k];
              if (!node_mask || node_mask[node[tg]]) s_y[sl][nt++] = tg;
            }
          }
        }
      }
      nt = __shfl_sync(0xffffffffu, nt, 0);
      __syncwarp();
      float om_part = 0.f;
      int bad = 0;
      for (int k = lane; k < nt; k += 32) {
        const int tg = s_y[sl][k];
        const int y = tok[tg];
        const float om = wr ? wr[tg] : (float)w[tg];
        bad |= (y < 0 || y >= V);
        s_y[sl][k] = y;
        s_om[sl][k] = om;
        om_part += om;
      }
      for (int o = 16; o > 0; o >>= 1) {
        om_part += __shfl_xor_sync(0xffffffffu, om_part, o);
        bad |= __shfl_xor_sync(0xffffffffu, bad, o);
      }
      if (lane == 0) {
        s_hdr[sl][0] = nt;
        s_hdr[sl][1] = bad;
        s_Om[sl] = om_part;
      }
      mbar_arrive_(&mfull[sl]);  // every lane, after its own writes of this slot
    }
    return;
  }
  // ============ compute warps ============
  int g = 0, it = 0;
  auto bar_c = [&]() { asm volatile("bar.sync 1, %0;" ::"n"(kPipeCompute) : "memory"); };
  for (int64_t row = row_begin + blockIdx.x; row < N; row += gridDim.x, ++it) {
    const int sl = it % kMetaSlots;
    mbar_wait_(&mfull[sl], (uint32_t)((it / kMetaSlots) & 1));
    const int nt = s_hdr[sl][0];
    const bool bad_any = s_hdr[sl][1] != 0;
    const float Omega = s_Om[sl];
    const int* ys = s_y[sl];
    const float* oms = s_om[sl];
    __nv_bfloat16* dx = dlogits + row * ld;
    // ---- pass 1 from the shared-memory ring (+ the target logits, read before anything is written) ----
    float m = -INFINITY, sum = 0.f;
    const bool live = Omega != 0.f && !bad_any;
    for (int c = 0; c < nchunk; ++c, ++g) {
      const int slot = g % kRing;
      mbar_wait_(&full[slot], (g / kRing) & 1);
      const int n = min(kChunkElems, V - c * kChunkElems);
      const uint4* src = reinterpret_cast<const uint4*>(ring + slot * kChunkElems);
      if (live) {
        // per thread and chunk: max of its elements on packed bf16 pairs, at most one rescale of the
        // running sum, then the sum of 2^(x log2e - m) with packed f32x2 FMAs / adds (the cluster
        // kernel's FAST pass 1, thread-local so no barrier per chunk)
        __nv_bfloat162 mx = __halves2bfloat162(__ushort_as_bfloat16((unsigned short)0xff80u),
                                               __ushort_as_bfloat16((unsigned short)0xff80u));
        for (int v = tid; v < n / 8; v += kPipeCompute) {
          const uint4 q = src[v];
          mx = __hmax2(__hmax2(mx, *reinterpret_cast<const __nv_bfloat162*>(&q.x)),
                       __hmax2(*reinterpret_cast<const __nv_bfloat162*>(&q.y), *reinterpret_cast<const __nv_bfloat162*>(&q.z)));
          mx = __hmax2(mx, *reinterpret_cast<const __nv_bfloat162*>(&q.w));
        }
        const float cm = fmaxf(__bfloat162float(mx.x), __bfloat162float(mx.y)) * kLog2e;
        if (cm > m) {
          sum *= ex2f(m - cm);  // m = -inf -> 0
          m = cm;
        }
        if (m != -INFINITY) {
          const float2 L2 = make_float2(kLog2e, kLog2e), NM = make_float2(-m, -m);
          float2 acc0 = make_float2(0.f, 0.f), acc1 = make_float2(0.f, 0.f);
          for (int v = tid; v < n / 8; v += kPipeCompute) {
            const uint4 q = src[v];
            const uint32_t in[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const float2 e2 = sm100::ffma2(bf2f(in[t]), L2, NM);
              const float2 e = make_float2(ex2f(e2.x), ex2f(e2.y));
              if (t & 1) acc1 = sm100::fadd2(acc1, e); else acc0 = sm100::fadd2(acc0, e);
            }
          }
          const float2 acc = sm100::fadd2(acc0, acc1);
          sum += acc.x + acc.y;
        }
        for (int k = tid; k < nt; k += kPipeCompute) {
          const int o = ys[k] - c * kChunkElems;
          if (o >= 0 && o < n) s_xy[k] = __bfloat162float(ring[slot * kChunkElems + o]);
        }
      }
      mbar_arrive_(&empty[slot]);  // every compute thread: its reads of this slot are done
    }
    if (!live) {
      Vec<16> z;
#pragma unroll
      for (int t = 0; t < 8; ++t) z.u[t] = 0u;
      for (int c = tid * 16; c < V; c += kPipeCompute * 16) st_vec<16>(dx + c, z);
      if (tid == 0) {
        const float lv = bad_any ? __int_as_float(0x7fc00000) : 0.f;
        if (bad_any && d_err) atomicExch(d_err, 1);
        ws_loss[row] = lv;
        ws_omega[row] = bad_any ? 0.f : Omega;
        if (tok_loss) tok_loss[row] = lv;
      }
      bar_c();  // every compute thread is done with metadata slot sl
      if (tid == 0) mbar_arrive_(&mfree[sl]);
      continue;
    }
    for (int o = 16; o > 0; o >>= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
      const float s2 = __shfl_xor_sync(0xffffffffu, sum, o);
      const float mm = fmaxf(m, m2);
      sum = (mm == -INFINITY) ? 0.f : sum * ex2f(m - mm) + s2 * ex2f(m2 - mm);
      m = mm;
    }
    if (lane == 0) { s_red[0][warp] = m; s_red[1][warp] = sum; }
    bar_c();
    if (tid == 0) {
      float M = -INFINITY, S = 0.f;
      for (int k = 0; k < kPipeCompute / 32; ++k) {
        const float m2 = s_red[0][k], s2 = s_red[1][k];
        const float mm = fmaxf(M, m2);
        S = (mm == -INFINITY) ? 0.f : S * ex2f(M - mm) + s2 * ex2f(m2 - mm);
        M = mm;
      }
      s_lse = M + log2f(S);
    }
    bar_c();
    const float lse2 = s_lse;
    float lpart = 0.f;
    for (int k = tid; k < nt; k += kPipeCompute) lpart += oms[k] * (lse2 * kLn2 - s_xy[k]);
    for (int o = 16; o > 0; o >>= 1) lpart += __shfl_xor_sync(0xffffffffu, lpart, o);
    bar_c();
    if (lane == 0) s_red[1][warp] = lpart;
    // ---- pass 2: re-read from L2, write dlogits ----
    const __nv_bfloat16* x = logits + row * ld;
    const float gO = gamma * Omega;
    const float2 L2 = make_float2(kLog2e, kLog2e), NL = make_float2(-lse2, -lse2), G2 = make_float2(gO, gO);
    auto softmax16 = [&](const Vec<16>& a, __nv_bfloat16* dst) {
      // packed f32x2 argument / scaling; 2 of every 8 pairs' exponentials as the degree-3 polynomial
      // on the FMA pipe (as the cluster kernel's pass 2: error far below the bf16 output rounding)
      Vec<16> o;
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const float2 a2 = sm100::ffma2(bf2f(a.u[t]), L2, NL);
        const float2 e = ((t & 3) == 3) ? sm100::exp2_poly2(a2) : make_float2(ex2f(a2.x), ex2f(a2.y));
        const float2 r2 = sm100::fmul2(e, G2);
        o.u[t] = f2bf(r2.x, r2.y);
      }
      st_vec<16>(dst, o);
    };
    constexpr int S2 = kPipeCompute * 16;
    constexpr int kMlp = 4;  // independent 32-byte L2 loads in flight per thread (4 / 8 / 12 measured equal)
    int c = tid * 16;
    for (; c + (kMlp - 1) * S2 < V; c += kMlp * S2) {
      Vec<16> a[kMlp];
#pragma unroll
      for (int u = 0; u < kMlp; ++u) a[u] = ld_last<16>(x + c + u * S2);
#pragma unroll
      for (int u = 0; u < kMlp; ++u) softmax16(a[u], dx + c + u * S2);
    }
    for (; c < V; c += S2) softmax16(ld_last<16>(x + c), dx + c);
    bar_c();
    for (int k = tid; k < nt; k += kPipeCompute) {
      const int y = ys[k];
      bool first = true;
      float om_y = 0.f;
      for (int k2 = 0; k2 < nt; ++k2) {
        if (ys[k2] == y) {
          if (k2 < k) first = false;
          om_y += oms[k2];
        }
      }
      if (first) {
        const float py = ex2f(fmaf(s_xy[k], kLog2e, -lse2));
        dx[y] = __float2bfloat16_rn(gamma * (Omega * py - om_y));
      }
    }
    if (tid == 0) {
      float L = 0.f;
      for (int k = 0; k < kPipeCompute / 32; ++k) L += s_red[1][k];
      ws_loss[row] = L;
      ws_omega[row] = Omega;
      if (tok_loss) tok_loss[row] = L;
    }
    bar_c();  // also: every compute thread is done with metadata slot sl and s_xy
    if (tid == 0) mbar_arrive_(&mfree[sl]);
  }
}

// fixed-order fp64 reduction of the per-row loss / Omega into sums[0..1]
__global__ void __launch_bounds__(1024) loss_sum_kernel(int64_t N, const float* __restrict__ ws_loss,
                                                        const float* __restrict__ ws_omega, double* __restrict__ sums) {
  const int64_t per = (N + blockDim.x - 1) / blockDim.x;
  const int64_t b0 = threadIdx.x * per, b1 = imin64(N, b0 + per);
  double a = 0.0, b = 0.0;
  for (int64_t i = b0; i < b1; ++i) { a += (double)ws_loss[i]; b += (double)ws_omega[i]; }
  __shared__ double sa[1024], sb[1024];
  sa[threadIdx.x] = a;
  sb[threadIdx.x] = b;
  __syncthreads();
  for (int w = 512; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) { sa[threadIdx.x] += sa[threadIdx.x + w]; sb[threadIdx.x] += sb[threadIdx.x + w]; }
    __syncthreads();
  }
  if (threadIdx.x == 0) { sums[0] = sa[0]; sums[1] = sb[0]; }
}

// ---------------------------------------------------------------------------------------------
// Cluster variant (V % 8 == 0, rows 16-byte aligned): a thread-block cluster of CS CTAs owns one row
// at a time; CTA c holds the c-th slice of Cq elements of the row in shared memory, so the row is
// read from HBM exactly once and written exactly once (4 V bytes / row, the §8(d) algorithmic
// traffic).  Per row: TMA bulk load of the slice (producer warp, NBUF-deep ring) -> pass 1 (max /
// sum-exp, own-slice target logits) -> the CS partials are exchanged through distributed shared
// memory (remote stores + remote mbarrier arrivals, no all-thread cluster barrier) -> pass 2
// overwrites the slice in shared memory with dlogits -> TMA bulk store (producer warp) while the
// compute warps already work on the next row.
// FAST passes (default): pass 1 = slice max on packed bf16 pairs (HMNMX2, no conversion), then the
// sum of 2^(x log2e - M) with packed f32x2 FMAs / adds (no online rescaling); pass 2 = packed f32x2
// exponent argument and gamma*Omega scaling.  ncu (r1e) counted ~17 issued instructions per logit
// for the online-rescaling passes; this form needs ~7.  25% of pass 2's exponentials run as a degree-3
// polynomial on the FMA pipe (relative error <= 7.5e-5 per term, far below the bf16 output rounding)
// to offload the MUFU unit; pass 1 stays on the MUFU so the lse keeps fp32 accuracy.
// ---------------------------------------------------------------------------------------------
#ifndef TT_LOSS_GROUP
#define TT_LOSS_GROUP 256
#endif
constexpr int kLcGroup = TT_LOSS_GROUP;            // threads per compute group
constexpr int kLcThreads = 2 * kLcGroup + 64;      // 2 compute groups + producer warp + meta warp
constexpr int kLcSlots = 4;                        // exchange slots (row it uses it % 4)

struct LcArgs {
  int64_t N;
  const __nv_bfloat16* logits;
  int64_t ld;
  int V, Cq, max_t;
  const int32_t* tok;
  const uint8_t* node_mask;
  int boundary_mode;
  float gamma;
  const int32_t* w;
  const float* wr;
  const int32_t *node, *node_start, *node_len, *succ_ptr, *succ_tok;
  __nv_bfloat16* dlogits;
  float *tok_loss, *ws_loss, *ws_omega;
  int32_t* d_err;
  int nocompute;  // development ablation (TT_DEV builds only) (TT_LOSS_NOCOMPUTE): stream the rows through without the math
};

__device__ __forceinline__ uint32_t lc_rank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ uint32_t lc_cid() { uint32_t r; asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r)); return r; }
__device__ __forceinline__ uint32_t lc_ncl() { uint32_t r; asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r)); return r; }
__device__ __forceinline__ uint32_t lc_mapa(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void lc_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void lc_wait_cluster(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                   smem_addr(b)),
               "r"(ph)
               : "memory");
}

// per-row metadata slot written by the meta warp: [nt, Omega, bad, pad] + y[max_t] + om[max_t] + xy[max_t]
struct LcMeta {
  int* hdr;
  int* y;
  float* om;
  float* xy;
};
__device__ __forceinline__ LcMeta lc_meta(uint8_t* base, int slot, int max_t) {
  uint8_t* p = base + (size_t)slot * (16 + (size_t)max_t * 12);
  LcMeta m;
  m.hdr = reinterpret_cast<int*>(p);
  m.y = reinterpret_cast<int*>(p + 16);
  m.om = reinterpret_cast<float*>(m.y + max_t);
  m.xy = m.om + max_t;
  return m;
}

// KPOLY: pairs (of 4 per 8-element vector) whose pass-2 exponentials run on the FMA pipe
template <int CS, int NBUF, int KPOLY, int KP1, int FAST = 0, int NG = 2>
__global__ void __launch_bounds__(kLcThreads, 1) loss_cluster_kernel(const LcArgs a) {
  // NG compute groups of GT threads (2 x 256: groups alternate rows; 1 x 512: one row at a time)
  constexpr int GT = 2 * kLcGroup / NG;
  extern __shared__ __align__(128) uint8_t lsm[];
  const int Cq = a.Cq;
  __nv_bfloat16* bufs = reinterpret_cast<__nv_bfloat16*>(lsm);                     // NBUF x Cq bf16
  float4* slots = reinterpret_cast<float4*>(lsm + (size_t)NBUF * Cq * 2);        // [kLcSlots][CS]
  uint64_t* full = reinterpret_cast<uint64_t*>(slots + kLcSlots * CS);           // [NBUF] slice loaded
  uint64_t* done = full + NBUF;                                                   // [NBUF] dlogits ready
  uint64_t* mfull = done + NBUF;                                                  // [NBUF] metadata ready
  uint64_t* mfree = mfull + NBUF;                                                 // [NBUF] metadata consumed
  uint64_t* xchg = mfree + NBUF;                                                  // [kLcSlots]
  uint8_t* meta_base = reinterpret_cast<uint8_t*>(xchg + kLcSlots);
  __shared__ float s_red[2][3][2 * kLcGroup / 32];
  __shared__ float s_max[2][2 * kLcGroup / 32];
  __shared__ float s_lse[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t cr = lc_rank();
  const int64_t row0 = lc_cid(), rstep = lc_ncl();
  const int off = (int)cr * Cq;
  const int n = max(0, min(Cq, a.V - off));  // elements of this CTA's slice (multiple of 8)
  if (tid == 0) {
    for (int k = 0; k < NBUF; ++k) {
      mbar_init_(&full[k], 1);
      mbar_init_(&done[k], 1);
      mbar_init_(&mfull[k], 1);
      mbar_init_(&mfree[k], 1);
    }
    for (int k = 0; k < kLcSlots; ++k) mbar_init_(&xchg[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  lc_cluster_sync();  // peers' barriers initialised before any remote arrival

  if (warp == 2 * kLcGroup / 32) {
    // ===================== producer warp: loads and stores of this CTA's slices =====================
    // Lane b < NBUF owns buffer b (rows it = b, b + NBUF, ...): a lane's bulk async-groups track only
    // its own buffer's store, so waiting for that store to have been read before reloading the
    // buffer never waits on another buffer's store.
    if (lane < NBUF) {
      const int b = lane;
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      auto load = [&](int64_t row) {
        if (n > 0) {
          mbar_expect_(&full[b], (uint32_t)n * 2);
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
                  smem_addr(bufs + (size_t)b * Cq)),
              "l"(a.logits + row * a.ld + off), "r"(n * 2), "r"(smem_addr(&full[b])), "l"(pol)
              : "memory");
        } else {
          mbar_arrive_(&full[b]);
        }
      };
      if (row0 + b * rstep < a.N) load(row0 + b * rstep);
      int it = b;
      for (int64_t row = row0 + b * rstep; row < a.N; row += (int64_t)NBUF * rstep, it += NBUF) {
        mbar_wait_(&done[b], (uint32_t)((it / NBUF) & 1));
        if (n > 0) {
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(
                           a.dlogits + row * a.ld + off),
                       "r"(smem_addr(bufs + (size_t)b * Cq)), "r"(n * 2), "l"(pol)
                       : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        const int64_t nrow = row + (int64_t)NBUF * rstep;
        if (nrow < a.N) {
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // this lane's slice b free again
          load(nrow);
        }
      }
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    __syncwarp();
    lc_cluster_sync();  // no CTA leaves while a peer may still write into its shared memory
    return;
  }
  if (warp == 2 * kLcGroup / 32 + 1) {
    // ===================== meta warp: targets / weights of upcoming rows (R7, R17, boundary) =====================
    int it = 0;
    for (int64_t row = row0; row < a.N; row += rstep, ++it) {
      const int b = it % NBUF;
      if (it >= NBUF) mbar_wait_(&mfree[b], (uint32_t)(((it / NBUF) - 1) & 1));
      LcMeta M = lc_meta(meta_base, b, a.max_t);
      int nt = 0;
      if (lane == 0) {
        const int32_t u = a.node[row];
        const bool last = row == (int64_t)a.node_start[u] + a.node_len[u] - 1;
        if (!last) {
          const int64_t tg = row + 1;
          if (!a.node_mask || a.node_mask[a.node[tg]]) { M.y[0] = (int)tg; nt = 1; }
        } else {
          const int sb = a.succ_ptr[u], se = a.succ_ptr[u + 1];
          if (!(a.boundary_mode == 1 && diverges(a.succ_tok, sb, se, a.w))) {
            for (int k = sb; k < se; ++k) {
              const int tg = a.succ_tok[k];
              if (!a.node_mask || a.node_mask[a.node[tg]]) M.y[nt++] = tg;
            }
          }
        }
      }
      nt = __shfl_sync(0xffffffffu, nt, 0);
      __syncwarp();
      float om_part = 0.f;
      int bad = 0;
      for (int k = lane; k < nt; k += 32) {
        const int tg = M.y[k];
        const int y = a.tok[tg];
        const float om = a.wr ? a.wr[tg] : (float)a.w[tg];
        bad |= (y < 0 || y >= a.V);
        M.y[k] = y;
        M.om[k] = om;
        om_part += om;
      }
      for (int o = 16; o > 0; o >>= 1) {
        om_part += __shfl_xor_sync(0xffffffffu, om_part, o);
        bad |= __shfl_xor_sync(0xffffffffu, bad, o);
      }
      __syncwarp();  // every lane's y / om writes happen-before lane 0's release below
      if (lane == 0) {
        M.hdr[0] = nt;
        reinterpret_cast<float*>(M.hdr)[1] = om_part;
        M.hdr[2] = bad;
        mbar_arrive_(&mfull[b]);  // release: the slot's writes above precede the arrival
      }
      __syncwarp();
    }
    lc_cluster_sync();
    return;
  }

  // ===================== compute groups: group g takes rows it = g, g + 2, ... =====================
  const int grp = warp / (GT / 32);
  const int gt = tid - grp * GT, gw = gt >> 5;
  auto bar_g = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "n"(GT) : "memory"); };
  int it = grp;
  for (int64_t row = row0 + grp * rstep; row < a.N; row += NG * rstep, it += NG) {
    const int b = it % NBUF;
    const int xs_slot = it % kLcSlots;
    mbar_wait_(&mfull[b], (uint32_t)((it / NBUF) & 1));
    LcMeta M = lc_meta(meta_base, b, a.max_t);
    if (kDevBuild && a.nocompute) {
      mbar_wait_(&full[b], (uint32_t)((it / NBUF) & 1));
      bar_g();
      if (gt == 0) {
        mbar_arrive_(&done[b]);
        mbar_arrive_(&mfree[b]);
      }
      continue;
    }
    const int nt = M.hdr[0];
    const float Omega = reinterpret_cast<const float*>(M.hdr)[1];
    const bool bad_any = M.hdr[2] != 0;
    // ---- pass 1 over this CTA's slice in shared memory ----
    mbar_wait_(&full[b], (uint32_t)((it / NBUF) & 1));
    __nv_bfloat16* xs = bufs + (size_t)b * Cq;
    const uint4* x4 = reinterpret_cast<const uint4*>(xs);
    float m = -INFINITY, sum = 0.f;
    float tx = 0.f;
    if constexpr (FAST) {
      // pass 1a: slice max on packed bf16 pairs (HMNMX2, no conversion); 1b: sum of 2^(x log2e - M)
      // with packed f32x2 FMAs / adds — no online rescaling, ~3 issue slots per element
      __nv_bfloat162 mx = __halves2bfloat162(__ushort_as_bfloat16((unsigned short)0xff80u),
                                             __ushort_as_bfloat16((unsigned short)0xff80u));
      for (int v = gt; v < n / 8; v += GT) {
        const uint4 q = x4[v];
        mx = __hmax2(__hmax2(mx, *reinterpret_cast<const __nv_bfloat162*>(&q.x)),
                     __hmax2(*reinterpret_cast<const __nv_bfloat162*>(&q.y), *reinterpret_cast<const __nv_bfloat162*>(&q.z)));
        mx = __hmax2(mx, *reinterpret_cast<const __nv_bfloat162*>(&q.w));
      }
      float tm = fmaxf(__bfloat162float(mx.x), __bfloat162float(mx.y));
      for (int o = 16; o > 0; o >>= 1) tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, o));
      if (lane == 0) s_max[grp][gw] = tm;
      if constexpr (FAST == 2) {
        // the target logits of this slice, read before pass 1b overwrites the slice (barrier below)
        for (int k = gt; k < nt; k += GT) {
          const int y = M.y[k];
          if (y >= off && y < off + n) {
            const float xy = __bfloat162float(xs[y - off]);
            M.xy[k] = xy;
            tx += M.om[k] * xy;
          }
        }
      }
      bar_g();
      tm = s_max[grp][0];
#pragma unroll
      for (int k = 1; k < GT / 32; ++k) tm = fmaxf(tm, s_max[grp][k]);
      m = tm * kLog2e;  // group max, log2 units
      if (m != -INFINITY) {
        const float2 L2 = make_float2(kLog2e, kLog2e), NM = make_float2(-m, -m);
        float2 acc0 = make_float2(0.f, 0.f), acc1 = make_float2(0.f, 0.f);
        uint4* xw4 = reinterpret_cast<uint4*>(xs);
        for (int v = gt; v < n / 8; v += GT) {
          const uint4 q = x4[v];
          const uint32_t in[4] = {q.x, q.y, q.z, q.w};
          uint32_t eh[4];
          (void)eh;
          (void)xw4;
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const float2 e2 = sm100::ffma2(bf2f(in[t]), L2, NM);
            const float2 e = (t >= 4 - KP1) ? sm100::exp2_poly2(e2) : make_float2(ex2f(e2.x), ex2f(e2.y));
            if (t & 1) acc1 = sm100::fadd2(acc1, e); else acc0 = sm100::fadd2(acc0, e);
            if constexpr (FAST == 2) eh[t] = f2h(e.x, e.y);
          }
          if constexpr (FAST == 2) xw4[v] = make_uint4(eh[0], eh[1], eh[2], eh[3]);  // e in place, fp16
        }
        const float2 acc = sm100::fadd2(acc0, acc1);
        sum = acc.x + acc.y;
      }
      for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    } else {
      for (int v = gt; v < n / 8; v += GT) {
        const uint4 q = x4[v];
        Vec<8> r;
        r.u[0] = q.x; r.u[1] = q.y; r.u[2] = q.z; r.u[3] = q.w;
        accum<8, KP1>(m, sum, r);
      }
      for (int o = 16; o > 0; o >>= 1) {
        const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
        const float s2 = __shfl_xor_sync(0xffffffffu, sum, o);
        const float mm = fmaxf(m, m2);
        sum = (mm == -INFINITY) ? 0.f : sum * ex2f(m - mm) + s2 * ex2f(m2 - mm);
        m = mm;
      }
    }
    // target logits that live in this slice (read before pass 2 overwrites them; FAST == 2 picked
    // them up before pass 1b)
    for (int k = gt; k < (FAST == 2 ? 0 : nt); k += GT) {
      const int y = M.y[k];
      if (y >= off && y < off + n) {
        const float xy = __bfloat162float(xs[y - off]);
        M.xy[k] = xy;
        tx += M.om[k] * xy;
      }
    }
    for (int o = 16; o > 0; o >>= 1) tx += __shfl_xor_sync(0xffffffffu, tx, o);
    if (lane == 0) { s_red[grp][0][gw] = m; s_red[grp][1][gw] = sum; s_red[grp][2][gw] = tx; }
    bar_g();
    if (gt == 0) {
      float Mx = -INFINITY, S = 0.f, TX = 0.f;
      for (int k = 0; k < GT / 32; ++k) {
        const float m2 = s_red[grp][0][k], s2 = s_red[grp][1][k];
        const float mm = fmaxf(Mx, m2);
        S = (mm == -INFINITY) ? 0.f : S * ex2f(Mx - mm) + s2 * ex2f(m2 - mm);
        Mx = mm;
        TX += s_red[grp][2][k];
      }
      // ---- exchange (M, S, TX) with the CS CTAs of the cluster through DSMEM ----
      // st.async: remote 16-byte store that completes as transaction bytes on the receiver's mbarrier
      // (no release/acquire fences on the critical path); each receiver arms CS x 16 bytes.
      const uint32_t my_slot = smem_addr(&slots[xs_slot * CS + cr]);
      const uint32_t my_bar = smem_addr(&xchg[xs_slot]);
#pragma unroll
      for (int c = 0; c < CS; ++c)
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                         lc_mapa(my_slot, (uint32_t)c)),
                     "f"(Mx), "f"(S), "f"(TX), "f"(0.f), "r"(lc_mapa(my_bar, (uint32_t)c))
                     : "memory");
      mbar_expect_(&xchg[xs_slot], (uint32_t)(CS * 16));
      mbar_wait_(&xchg[xs_slot], (uint32_t)((it / kLcSlots) & 1));
      float GM = -INFINITY, GS = 0.f, GT = 0.f;
      for (int c = 0; c < CS; ++c) {
        const float4 sv = slots[xs_slot * CS + c];
        const float mm = fmaxf(GM, sv.x);
        GS = (mm == -INFINITY) ? 0.f : GS * ex2f(GM - mm) + sv.y * ex2f(sv.x - mm);
        GM = mm;
        GT += sv.z;
      }
      const float lse2 = GM + log2f(GS);
      s_lse[grp] = lse2;
      if (cr == 0) {
        const float lv = bad_any ? __int_as_float(0x7fc00000) : (Omega == 0.f ? 0.f : Omega * lse2 * kLn2 - GT);
        if (bad_any && a.d_err) atomicExch(a.d_err, 1);
        a.ws_loss[row] = lv;
        a.ws_omega[row] = bad_any ? 0.f : Omega;
        if (a.tok_loss) a.tok_loss[row] = lv;
      }
    }
    bar_g();
    const float lse2 = s_lse[grp];
    const float gO = bad_any ? 0.f : a.gamma * Omega;
    // ---- pass 2: dlogits = gamma Omega softmax, in place in shared memory ----
    uint4* y4 = reinterpret_cast<uint4*>(xs);
    if constexpr (FAST == 2) {
      // the slice holds e = 2^(x log2e - m) (fp16, pass 1b): softmax = e 2^(m - lse2), one multiply
      // per element and no exponential (the MUFU work of the row halves); fp16 keeps 11 significant
      // bits (relative 2^-11, below the bf16 output rounding; values under 2^-24 flush to 0, an
      // absolute error < 6e-8 gamma Omega)
      const float sc = (m == -INFINITY) ? 0.f : gO * ex2f(m - lse2);
      const float2 S2 = make_float2(sc, sc);
      for (int v = gt; v < n / 8; v += GT) {
        const uint4 q = y4[v];
        const uint32_t in[4] = {q.x, q.y, q.z, q.w};
        uint32_t o[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const float2 r2 = sm100::fmul2(__half22float2(*reinterpret_cast<const __half2*>(&in[t])), S2);
          o[t] = f2bf(r2.x, r2.y);
        }
        y4[v] = make_uint4(o[0], o[1], o[2], o[3]);
      }
    } else if constexpr (FAST) {
      const float2 L2 = make_float2(kLog2e, kLog2e), NL = make_float2(-lse2, -lse2), G2 = make_float2(gO, gO);
      for (int v = gt; v < n / 8; v += GT) {
        const uint4 q = y4[v];
        const uint32_t in[4] = {q.x, q.y, q.z, q.w};
        uint32_t o[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const float2 a2 = sm100::ffma2(bf2f(in[t]), L2, NL);
          const float2 e = (t >= 4 - KPOLY) ? sm100::exp2_poly2(a2) : make_float2(ex2f(a2.x), ex2f(a2.y));
          const float2 r2 = sm100::fmul2(e, G2);
          o[t] = f2bf(r2.x, r2.y);
        }
        y4[v] = make_uint4(o[0], o[1], o[2], o[3]);
      }
    } else
    for (int v = gt; v < n / 8; v += GT) {
      const uint4 q = y4[v];
      const uint32_t in[4] = {q.x, q.y, q.z, q.w};
      uint32_t o[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const float2 f = bf2f(in[t]);
        if (t >= 4 - KPOLY) {  // part of the exponentials on the FMA pipe (degree-3 polynomial, rel. err ~1e-4 << bf16)
          const float2 e = sm100::exp2_poly2(sm100::ffma2(f, make_float2(kLog2e, kLog2e), make_float2(-lse2, -lse2)));
          o[t] = f2bf(gO * e.x, gO * e.y);
        } else {
          o[t] = f2bf(gO * ex2f(fmaf(f.x, kLog2e, -lse2)), gO * ex2f(fmaf(f.y, kLog2e, -lse2)));
        }
      }
      y4[v] = make_uint4(o[0], o[1], o[2], o[3]);
    }
    bar_g();
    // ---- fix-up of the target entries of this slice: gamma (Omega p_y - sum_{k: y_k = y} omega_k) ----
    if (!bad_any) {
      for (int k = gt; k < nt; k += GT) {
        const int y = M.y[k];
        if (y < off || y >= off + n) continue;
        bool first = true;
        float om_y = 0.f;
        for (int k2 = 0; k2 < nt; ++k2) {
          if (M.y[k2] == y) {
            if (k2 < k) first = false;
            om_y += M.om[k2];
          }
        }
        if (first) {
          const float py = ex2f(fmaf(M.xy[k], kLog2e, -lse2));
          xs[y - off] = __float2bfloat16_rn(a.gamma * (Omega * py - om_y));
        }
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> TMA store
    bar_g();
    if (gt == 0) {
      mbar_arrive_(&done[b]);
      mbar_arrive_(&mfree[b]);
    }
  }
  lc_cluster_sync();
}

template <int CS, int NBUF>
size_t lc_smem(int Cq, int max_t) {
  return (size_t)NBUF * Cq * 2 + kLcSlots * CS * 16 + (4 * NBUF + kLcSlots) * 8 + (size_t)NBUF * (16 + (size_t)max_t * 12);
}

// The 4-CTA clusters do not tile every SM (GPCs whose SM count is not a multiple of 4: 33 clusters
// = 132 of 148 SMs on B200).  The SMs they leave idle run loss_pipe_kernel (one CTA per SM, one row
// at a time) over the tail rows on a side stream forked from and joined back into the caller's
// stream; the row split follows the two kernels' measured per-SM row rates.
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  SideStream() = default;
  SideStream(const SideStream&) = delete;
  SideStream& operator=(const SideStream&) = delete;
  SideStream(SideStream&& o) noexcept : s(o.s), fork(o.fork), join(o.join) { o.s = nullptr; o.fork = o.join = nullptr; }
  SideStream& operator=(SideStream&& o) noexcept {
    std::swap(s, o.s); std::swap(fork, o.fork); std::swap(join, o.join);
    return *this;
  }
  ~SideStream() {
    // thread exit: release the side stream and its events (work still queued on them completes
    // first: cudaStreamDestroy / cudaEventDestroy defer the release; errors at teardown ignored)
    if (join) cudaEventDestroy(join);
    if (fork) cudaEventDestroy(fork);
    if (s) cudaStreamDestroy(s);
    cudaGetLastError();
  }
};
SideStream* side_stream(cudaStream_t st) {
  thread_local std::unordered_map<int, SideStream> per_dev;
  int dev = 0;
  cudaGetDevice(&dev);
  SideStream& ss = per_dev[dev];
  if (!ss.s) {
    // never create resources inside a stream capture (the first call on this thread/device then
    // runs without the split; later captures reuse the stream and events made outside)
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
      cudaGetLastError();
      return nullptr;
    }
    if (cudaStreamCreateWithFlags(&ss.s, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ss.join, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      ss = SideStream{};  // the moved-from temporary releases whatever was created
      return nullptr;
    }
  }
  return &ss;
}

// Outcome of a cluster launch attempt: kNotLaunched leaves the stream untouched (the caller may try
// another kernel); once the cluster kernel is enqueued the attempt is final (kLaunched / kFailed), so
// a failure after that point is reported, never retried over rows that may already hold dlogits
// (in-place mode).
enum class LcLaunch { kNotLaunched, kLaunched, kFailed };

template <int CS, int NBUF, int KPOLY = 1, int KP1 = 0, int FAST = 0, int NG = 2>
LcLaunch try_launch_cluster(const LcArgs& a0, int sms, cudaStream_t st) {
  LcArgs a = a0;
  a.Cq = ((a.V + CS - 1) / CS + 7) / 8 * 8;
  const size_t smem = lc_smem<CS, NBUF>(a.Cq, a.max_t);
  if (smem + 1024 > 232448) return LcLaunch::kNotLaunched;  // static shared memory + margin
  auto kern = loss_cluster_kernel<CS, NBUF, KPOLY, KP1, FAST, NG>;
  cudaGetLastError();  // a stale error of an earlier call must not be taken for this launch's
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    cudaGetLastError();
    return LcLaunch::kNotLaunched;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(CS * std::max(1, sms / CS)));
  cfg.blockDim = dim3(kLcThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int ncl = 0;
  if (cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg) != cudaSuccess || ncl <= 0) {
    cudaGetLastError();
    return LcLaunch::kNotLaunched;
  }
  int64_t want = std::min<int64_t>((int64_t)ncl, a.N);
  if (const char* mc = dev_getenv("TT_LOSS_MAXCL")) want = std::min<int64_t>(want, std::max(1, atoi(mc)));  // dev: SM-count sweep
  if (dev_getenv("TT_LOSS_DEBUG")) fprintf(stderr, "loss_cluster<%d,%d>: %d active clusters, Cq %d, smem %zu\n", CS, NBUF, ncl, a.Cq, smem);
  cfg.gridDim = dim3((unsigned)(want * CS));
  // tail rows for the SMs the clusters leave idle (split by per-SM row rate, pipe / cluster ~ 0.75:
  // profiles/r1k_loss_split.txt, re-swept in profiles/r2d_loss_split.txt)
  const int idle = sms - (int)want * CS;
  double ratio = 0.75;
  if (const char* e = dev_getenv("TT_LOSS_SPLIT")) ratio = atof(e);  // development A/B: 0 disables the split
  int64_t n_pipe = 0;
  if (idle > 0 && ratio > 0 && a.N >= 8 * sms && (a.V % 16 == 0) && (a.ld % 16 == 0) &&
      ((reinterpret_cast<uintptr_t>(a.logits) | reinterpret_cast<uintptr_t>(a.dlogits)) % 32 == 0))
    n_pipe = (int64_t)((double)a.N * idle * ratio / ((double)want * CS + idle * ratio));
  SideStream* ss = n_pipe > 0 ? side_stream(st) : nullptr;
  if (ss && cudaFuncSetAttribute(loss_pipe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPipeSmem) != cudaSuccess) {
    cudaGetLastError();
    ss = nullptr;
  }
  if (!ss) n_pipe = 0;
  const int64_t N = a.N;
  a.N = N - n_pipe;
  if (ss && cudaEventRecord(ss->fork, st) != cudaSuccess) {
    cudaGetLastError();
    ss = nullptr;
    n_pipe = 0;
    a.N = N;
  }
  if (cudaLaunchKernelEx(&cfg, kern, a) != cudaSuccess) {
    cudaGetLastError();
    if (!ss) return LcLaunch::kNotLaunched;
    // the fork event was recorded on st: keep the side stream joined (capture stays balanced)
    cudaStreamWaitEvent(ss->s, ss->fork, 0);
    cudaEventRecord(ss->join, ss->s);
    cudaStreamWaitEvent(st, ss->join, 0);
    return LcLaunch::kNotLaunched;
  }
  count_launch();
  LcLaunch res = LcLaunch::kLaunched;
  if (ss) {
    // launched after the clusters so its CTAs land on the SMs they left free
    cudaStreamWaitEvent(ss->s, ss->fork, 0);
    loss_pipe_kernel<<<(unsigned)idle, kPipeThreads, kPipeSmem, ss->s>>>(
        N, a.logits, a.ld, a.V, a.tok, a.node_mask, a.boundary_mode, a.gamma, a.w, a.wr, a.node, a.node_start,
        a.node_len, a.succ_ptr, a.succ_tok, a.dlogits, a.tok_loss, a.ws_loss, a.ws_omega, a.d_err, N - n_pipe);
    const cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) {
      count_launch();
    } else {
      set_error("loss_pipe_kernel (tail rows %lld..%lld): %s", (long long)(N - n_pipe), (long long)N, cudaGetErrorString(e));
      res = LcLaunch::kFailed;
    }
    // always join, even after a failed tail launch
    cudaEventRecord(ss->join, ss->s);
    cudaStreamWaitEvent(st, ss->join, 0);
  }
  return res;
}

}  // namespace

tt_status launch_loss_sums(int64_t N, const float* ws_loss, const float* ws_omega, double* sums, cudaStream_t st) {
  loss_sum_kernel<<<1, 1024, 0, st>>>(N, ws_loss, ws_omega, sums);
  count_launch();
  return check_launch("loss_sum_kernel");
}

tt_status launch_loss(const tt_packed& pk, const __nv_bfloat16* logits, int64_t ld, int vocab, const int32_t* tok,
                      const uint8_t* node_mask, int boundary_mode, float gamma, __nv_bfloat16* dlogits, float* tok_loss,
                      double* sums, int32_t* d_err, float* ws_loss, float* ws_omega, cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // 1 CTA (1024 threads) per SM: 148 rows (~44 MB at V = 151,936) in flight, so pass 2 re-reads from L2
  const int64_t grid = std::min<int64_t>(pk.n_tokens, (int64_t)sms);
  // loss_pipe_kernel: 16-element vectors over whole rows (V % 16 == 0) and 32-byte aligned rows
  const bool v16 = (vocab % 16 == 0) && (ld % 16 == 0) &&
                   ((reinterpret_cast<uintptr_t>(logits) | reinterpret_cast<uintptr_t>(dlogits)) % 32 == 0);
  LcLaunch lc = LcLaunch::kNotLaunched;
  if (vocab % 8 == 0) {
    LcArgs a{pk.n_tokens, logits, ld, vocab, 0, 0, tok, node_mask, boundary_mode, gamma, pk.w, pk.wr,
             pk.node, pk.node_start, pk.node_len, pk.succ_ptr, pk.succ_tok, dlogits, tok_loss, ws_loss, ws_omega, d_err, 0};
    a.max_t = std::max(1, pk.max_succ);
    // shipped kernel: 4-CTA clusters x 3 buffers, FAST passes, 25% polynomial exponentials in pass 2
    // only (25% in pass 1 too was ~1% faster, but its 7.5e-5 relative error per term moves the lse by
    // up to ~2e-5 and broke the dlogits tolerance on a small-vocabulary random case); 2 buffers when
    // many continuation targets do not leave room for 3.  Dev variant 25 keeps pass 1's exponentials
    // in place as fp16 so pass 2 needs no exponential: 1-3.5% faster (profiles/r2_loss_fp16_ab.txt),
    // but the fp16 intermediate (2^-11 relative) pushes dlogits across a bf16 rounding boundary
    // (1 element in 600K at V = 1000 missed the 2^-8 |dx| bound), so it is not shipped.
    int variant = 21;
#ifdef TT_DEV
    // development A/B: 0 ring/L2 kernel, 1 CS4x3, 3 CS8x4, 1x: poly splits, 2x: FAST passes, 3x: other
    // cluster sizes; TT_LOSS_NOCOMPUTE streams the rows through without the math
    if (const char* e = dev_getenv("TT_LOSS_VARIANT")) variant = atoi(e);
    a.nocompute = dev_getenv("TT_LOSS_NOCOMPUTE") ? 1 : 0;
    if (variant == 0) lc = LcLaunch::kNotLaunched;
    else if (variant == 1) lc = try_launch_cluster<4, 3>(a, sms, st);
    else if (variant == 11) lc = try_launch_cluster<4, 3, 2, 0>(a, sms, st);
    else if (variant == 12) lc = try_launch_cluster<4, 3, 2, 1>(a, sms, st);
    else if (variant == 13) lc = try_launch_cluster<4, 3, 1, 1>(a, sms, st);
    else if (variant == 25) lc = try_launch_cluster<4, 3, 0, 0, 2>(a, sms, st);
    else if (variant == 22) lc = try_launch_cluster<4, 3, 2, 0, 1>(a, sms, st);
    else if (variant == 23) lc = try_launch_cluster<4, 3, 2, 1, 1>(a, sms, st);
    else if (variant == 24) lc = try_launch_cluster<4, 3, 1, 1, 1>(a, sms, st);
    else if (variant == 26) lc = try_launch_cluster<4, 3, 1, 1, 1, 1>(a, sms, st);
    else if (variant == 31) lc = try_launch_cluster<8, 5, 1, 1, 1>(a, sms, st);
    else if (variant == 32) lc = try_launch_cluster<8, 4, 1, 1, 1>(a, sms, st);
    else if (variant == 33) lc = try_launch_cluster<2, 1, 1, 1, 1>(a, sms, st);
    else if (variant == 34) lc = try_launch_cluster<8, 5, 2, 1, 1>(a, sms, st);
    else if (variant == 35) lc = try_launch_cluster<3, 2, 1, 1, 1>(a, sms, st);
    else if (variant == 36) lc = try_launch_cluster<6, 4, 1, 1, 1>(a, sms, st);
    else if (variant == 3) lc = try_launch_cluster<8, 4>(a, sms, st);
#endif
    if (variant == 21) lc = try_launch_cluster<4, 3, 1, 0, 1>(a, sms, st);
    if (variant != 0 && lc == LcLaunch::kNotLaunched) lc = try_launch_cluster<4, 2, 1, 0, 1>(a, sms, st);
  }
  if (lc == LcLaunch::kFailed) return TT_ERR_CUDA;  // message set by try_launch_cluster
  if (lc == LcLaunch::kNotLaunched) {
    if (v16) {
      const size_t smem = kPipeSmem;
      if (cudaFuncSetAttribute(loss_pipe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
        set_error("loss_pipe_kernel: smem attribute: %s", cudaGetErrorString(cudaGetLastError()));
        return TT_ERR_CUDA;
      }
      loss_pipe_kernel<<<(unsigned)std::min<int64_t>(pk.n_tokens, sms), kPipeThreads, smem, st>>>(
          pk.n_tokens, logits, ld, vocab, tok, node_mask, boundary_mode, gamma, pk.w, pk.wr, pk.node, pk.node_start,
          pk.node_len, pk.succ_ptr, pk.succ_tok, dlogits, tok_loss, ws_loss, ws_omega, d_err, (int64_t)0);
    } else {
      loss_kernel<8><<<(unsigned)grid, kLossThreads, 0, st>>>(pk.n_tokens, logits, ld, vocab, tok, node_mask, boundary_mode,
                                                              gamma, pk.w, pk.wr, pk.node, pk.node_start, pk.node_len,
                                                              pk.succ_ptr, pk.succ_tok, dlogits, tok_loss, ws_loss,
                                                              ws_omega, d_err);
    }
    count_launch();
    tt_status s = check_launch("loss_kernel");
    if (s) return s;
  }
  loss_sum_kernel<<<1, 1024, 0, st>>>(pk.n_tokens, ws_loss, ws_omega, sums);
  count_launch();
  return check_launch("loss_sum_kernel");
}

}  // namespace tt
