// gemm_sm100.cu — the LM-head contractions of NEXT-f3 (the "gradient scaling step
// before the backward propagation") as one hand-written sm_100a GEMM with fused epilogues.
//
//   D[M, N] = A[M, K] . B[K, N]      bf16 operands, fp32 accumulation in TMEM
//
// Design: a CTA pair (thread-block cluster of 2, tcgen05 cta_group::2) owns a 256 x 256 output tile;
// each CTA stages its 128 rows of A and its 128 columns of B per 64-deep K step (TMA, SWIZZLE_128B,
// 6-stage ring, 32 KB / stage / CTA), the leader CTA's MMA warp issues the M = 256, N = 256 UMMA
// that reads both CTAs' shared memory, and each CTA's 128 accumulator rows live in its own TMEM
// (two 256-column buffers: the epilogue of tile i overlaps the main loop of tile i + 1).
// Persistent: one pair per two SMs, tiles strided over the pairs, M fastest so concurrently running
// pairs share their B tiles in L2.  Operands may be K-major or MN-major (the LM head needs
// H W^T, G W and G^T H), read through 2-D tensor maps; out-of-range rows / columns / K are zero-filled
// by TMA and masked in the epilogue.
//
// Epilogues (8 warps per CTA, one accumulator row and 128 columns per thread):
//   kEpiLsePartial  sweep 1 of the restoration CE: per row and 128-column slice, the (max, sum-exp)
//                   partial of x log2(e) (columns >= vocab masked), and the logits of the row's
//                   targets that fall in the slice — the [N, V] logits are never stored
//   kEpiDlogits     sweep 2: G = gamma (Omega 2^(x log2e - lse2) - sum_{k: y_k = col} omega_k) in bf16
//   kEpiStoreBF16   plain store (dW)
//   kEpiAccF32      fp32 store or accumulate into global (dH across vocabulary chunks)
#include <cudaTypedefs.h>

#include <algorithm>

#include "sm100_ptx.cuh"
#include "tt_internal.cuh"

namespace tt {
namespace gemm {
namespace {

using namespace sm100;

constexpr int kBK = 64;
constexpr int kStages = 6;
constexpr uint32_t kHalfBytes = 128 * kBK * 2;        // 16 KB: 128 rows x 64 K of one operand, one CTA
constexpr uint32_t kStageBytes = 2 * kHalfBytes;      // A half + B half
constexpr int kEpiWarps = 8;
constexpr int kThreads = 32 * (2 + kEpiWarps);
constexpr uint32_t kOffBar = kStages * kStageBytes;   // 192 KB of stages
constexpr uint32_t kSmemBytes = kOffBar + 256;
static_assert(kSmemBytes <= 232448, "GEMM exceeds 227 KB of shared memory");
constexpr uint32_t kPeerMask = 0xFEFFFFFFu;           // shared::cluster address -> the leader CTA's copy
constexpr int kGemmWaitDefault = 0;

struct Args {
  int M, N, K;
  int a_mn, b_mn;          // operand majors (0: K contiguous, 1: M / N contiguous)
  int tiles_m, tiles_n;
  void* out;               // bf16 / fp32 [M, ldo] row-major
  int64_t ldo;
  int beta;                // kEpiAccF32: accumulate into out
  // cross-entropy epilogues (columns are vocabulary ids col_offset + n)
  int col_offset, vocab;
  float2* part;            // [2 tiles_n][M] (max, sum-exp) in log2 units
  int max_t;               // targets per row capacity
  const int* tgt_cnt;      // [M]
  const int* tgt_y;        // [M, max_t] distinct target ids of the row
  const float* tgt_w;      // [M, max_t] summed weight of each distinct target
  float* tgt_x;            // [M, max_t] the target logits (written by the slice holding y)
  const float* lse2;       // [M] log2-domain lse (kEpiDlogits)
  const float* g_omega;    // [M] gamma * Omega (0 for rows without a prediction)
  float gamma;
  int wait_mode;           // dev A/B (TT_GEMM_WAIT): 0 spin try_wait, 1 suspend-time hint, 2 nanosleep back-off
};

// barrier wait of the long-waiting roles (epilogue for the accumulator, producer for a free stage)
__device__ __forceinline__ void wait_long(const Args& p, uint64_t* bar, uint32_t parity) {
  const int m = kDevBuild ? p.wait_mode : kGemmWaitDefault;
  if (m == 1) mbar_wait_hint(bar, parity, 20000);
  else if (m == 2) mbar_wait_sleep(bar, parity);
  else mbar_wait(bar, parity);
}

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t n_clusters() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// 2-D TMA load issued by either CTA of the pair; completion bytes land on the LEADER's barrier
__device__ __forceinline__ void tma_load_2sm(uint32_t dst, const CUtensorMap* m, uint32_t bar_leader, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, 0, "
      "%4}], [%2];" ::"r"(dst),
      "l"(m), "r"(bar_leader), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void mma_pair(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// arrive on the barrier at this offset in BOTH CTAs once the pair's issued MMAs have completed
__device__ __forceinline__ void commit_pair(uint64_t* bar) {
  asm volatile(
      "{\n.reg .pred e;\n.reg .b16 m;\nmov.b16 m, 3;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n}\n" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void arrive_leader(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(smem_u32(bar) & kPeerMask) : "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

template <int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, const Args p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  if (smem_u32(smem) & 1023u) __trap();
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kOffBar);   // [kStages] (leader's count)
  uint64_t* empty = full + kStages;                                // [kStages] (each CTA's own)
  uint64_t* acc_full = empty + kStages;                            // [2]
  uint64_t* acc_empty = acc_full + 2;                              // [2] (leader's count)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cta_rank();
  const bool leader = rank == 0;
  const int pair = (int)cluster_id(), npairs = (int)n_clusters();
  const int n_tiles = p.tiles_m * p.tiles_n;
  const int nk = (p.K + kBK - 1) / kBK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 2 * kEpiWarps);
    }
    mbar_fence_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // both CTAs' barriers and TMEM exist before any remote arrival or pair MMA
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ===================== TMA producer (both CTAs) =====================
    if (lane == 0) {
      tma_prefetch(&tmA);
      tma_prefetch(&tmB);
      const uint32_t sbase = smem_u32(smem);
      int it = 0;
      for (int tile = pair; tile < n_tiles; tile += npairs) {
        const int tm = tile % p.tiles_m, tn = tile / p.tiles_m;
        const int m0 = tm * 256 + 128 * (int)rank, n0 = tn * 256 + 128 * (int)rank;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % kStages;
          if (it >= kStages) wait_long(p, &empty[s], ((it / kStages) - 1) & 1);
          if (leader) expect_tx(&full[s], 2 * kStageBytes);
          const uint32_t fb = smem_u32(&full[s]) & kPeerMask;
          const uint32_t a_dst = sbase + s * kStageBytes, b_dst = a_dst + kHalfBytes;
          const int k0 = kb * kBK;
          if (p.a_mn) {
            tma_load_2sm(a_dst, &tmA, fb, m0, k0);
            tma_load_2sm(a_dst + kHalfBytes / 2, &tmA, fb, m0 + 64, k0);
          } else {
            tma_load_2sm(a_dst, &tmA, fb, k0, m0);
          }
          if (p.b_mn) {
            tma_load_2sm(b_dst, &tmB, fb, n0, k0);
            tma_load_2sm(b_dst + kHalfBytes / 2, &tmB, fb, n0 + 64, k0);
          } else {
            tma_load_2sm(b_dst, &tmB, fb, k0, n0);
          }
        }
      }
      // tail: every stage's last use has been released by the pair's MMAs (their multicast commits
      // land on this CTA's barriers) before the CTA may retire
      for (int j = std::max(0, it - kStages); j < it; ++j) mbar_wait(&empty[j % kStages], (j / kStages) & 1);
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (leader CTA, whole warp, one elected lane) =====================
    if (leader) {
      // K-major operand: 128 rows x 128 B, 8-row atoms of 1024 B (SBO); per K=16 step +32 B.
      // MN-major operand: two 64-wide MN groups of 64 K rows (LBO = 8 KB), 8-row K groups (SBO =
      // 1024 B); per K=16 step +16 rows x 128 B = 2 KB.
      const uint32_t idesc = idesc_bf16(256, 256, p.a_mn, p.b_mn);
      const uint32_t sbase = warp_uniform(smem_u32(smem));
      const uint32_t tm0 = warp_uniform(tmem);
      int it = 0, tc = 0;
      for (int tile = pair; tile < n_tiles; tile += npairs, ++tc) {
        const int b = tc & 1;
        if (tc >= 2) mbar_wait(&acc_empty[b], ((tc >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t d_tmem = tm0 + 256 * b;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % kStages;
          mbar_wait(&full[s], (it / kStages) & 1);
          tc_fence_after();
          const uint32_t a_s = sbase + s * kStageBytes, b_s = a_s + kHalfBytes;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t ad = p.a_mn ? sdesc(a_s + kk * 2048, kHalfBytes / 2, 1024) : sdesc(a_s + kk * 32, 16, 1024);
            const uint64_t bd = p.b_mn ? sdesc(b_s + kk * 2048, kHalfBytes / 2, 1024) : sdesc(b_s + kk * 32, 16, 1024);
            mma_pair(d_tmem, ad, bd, idesc, (kb > 0 || kk > 0) ? 1u : 0u);
          }
          commit_pair(&empty[s]);
        }
        commit_pair(&acc_full[b]);
      }
    }
  } else {
    // ===================== epilogue warps (both CTAs) =====================
    const int q = warp & 3;                 // TMEM lane quadrant this warp may access
    const int half = (warp - 2) >> 2;       // 128-column half of the tile
    const int rl = q * 32 + lane;           // accumulator row (TMEM lane)
    const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
    int tc = 0;
    for (int tile = pair; tile < n_tiles; tile += npairs, ++tc) {
      const int b = tc & 1;
      const int tm = tile % p.tiles_m, tn = tile / p.tiles_m;
      const int row = tm * 256 + 128 * (int)rank + rl;
      const int c_base = tn * 256 + 128 * half;          // first column of this thread's 128
      const bool rv = row < p.M;
      wait_long(p, &acc_full[b], (tc >> 1) & 1);
      tc_fence_after();
      float m_run = -INFINITY, s_run = 0.f;
      int nt = 0;
      float g_om = 0.f, l2 = 0.f;
      if constexpr (EPI == kEpiLsePartial || EPI == kEpiDlogits) {
        if (rv) nt = p.tgt_cnt[row];
      }
      if constexpr (EPI == kEpiDlogits) {
        if (rv) { g_om = p.g_omega[row]; l2 = p.lse2[row]; }
      }
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t v[32];
        tmem_ld32(tl + 256 * b + 128 * half + 32 * c, v);
        tmem_wait_ld();
        const int col0 = c_base + 32 * c;    // GEMM column of v[0]
        if constexpr (EPI == kEpiLsePartial) {
          // vocabulary columns >= vocab (TMA zero fill) do not exist
          const int lim = p.vocab - p.col_offset - col0;
          float cm = -INFINITY;
#pragma unroll
          for (int u = 0; u < 32; ++u) {
            const float x = __uint_as_float(v[u]) * kLog2e;
            v[u] = __float_as_uint(u < lim ? x : -INFINITY);
            cm = fmaxf(cm, __uint_as_float(v[u]));
          }
          if (cm > m_run) {
            s_run *= ex2(m_run - cm);
            m_run = cm;
          }
          if (m_run != -INFINITY) {
            float a0 = 0.f, a1 = 0.f;
#pragma unroll
            for (int u = 0; u < 32; u += 2) {
              a0 += ex2(__uint_as_float(v[u]) - m_run);
              a1 += ex2(__uint_as_float(v[u + 1]) - m_run);
            }
            s_run += a0 + a1;
          }
          for (int k = 0; k < nt; ++k) {
            const int y = p.tgt_y[(int64_t)row * p.max_t + k] - p.col_offset - col0;
            if (y >= 0 && y < 32) {
              float xv = 0.f;
#pragma unroll
              for (int u = 0; u < 32; ++u) xv = (u == y) ? __uint_as_float(v[u]) : xv;
              p.tgt_x[(int64_t)row * p.max_t + k] = xv * kLn2;  // back to natural units
            }
          }
        } else if constexpr (EPI == kEpiDlogits) {
          uint32_t o[16];
#pragma unroll
          for (int u = 0; u < 32; u += 2) {
            const float2 e = make_float2(ex2(fmaf(__uint_as_float(v[u]), kLog2e, -l2)),
                                         ex2(fmaf(__uint_as_float(v[u + 1]), kLog2e, -l2)));
            v[u] = __float_as_uint(g_om * e.x);
            v[u + 1] = __float_as_uint(g_om * e.y);
          }
          for (int k = 0; k < nt; ++k) {
            const int y = p.tgt_y[(int64_t)row * p.max_t + k] - p.col_offset - col0;
            if (y >= 0 && y < 32) {
              const float wy = p.gamma * p.tgt_w[(int64_t)row * p.max_t + k];
#pragma unroll
              for (int u = 0; u < 32; ++u)
                if (u == y) v[u] = __float_as_uint(__uint_as_float(v[u]) - wy);
            }
          }
#pragma unroll
          for (int u = 0; u < 16; ++u) o[u] = pack_bf16(__uint_as_float(v[2 * u]), __uint_as_float(v[2 * u + 1]));
          if (rv) {
            __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(p.out) + (int64_t)row * p.ldo + col0;
            if (col0 + 32 <= p.N && ((p.ldo & 7) == 0)) {
#pragma unroll
              for (int u = 0; u < 4; ++u)
                reinterpret_cast<uint4*>(dst)[u] = make_uint4(o[4 * u], o[4 * u + 1], o[4 * u + 2], o[4 * u + 3]);
            } else {
#pragma unroll
              for (int u = 0; u < 32; ++u)
                if (col0 + u < p.N) dst[u] = __ushort_as_bfloat16((unsigned short)((o[u >> 1] >> (16 * (u & 1))) & 0xffffu));
            }
          }
        } else if constexpr (EPI == kEpiStoreBF16) {
          if (rv) {
            uint32_t o[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) o[u] = pack_bf16(__uint_as_float(v[2 * u]), __uint_as_float(v[2 * u + 1]));
            __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(p.out) + (int64_t)row * p.ldo + col0;
            if (col0 + 32 <= p.N && ((p.ldo & 7) == 0)) {
#pragma unroll
              for (int u = 0; u < 4; ++u)
                reinterpret_cast<uint4*>(dst)[u] = make_uint4(o[4 * u], o[4 * u + 1], o[4 * u + 2], o[4 * u + 3]);
            } else {
#pragma unroll
              for (int u = 0; u < 32; ++u)
                if (col0 + u < p.N) dst[u] = __ushort_as_bfloat16((unsigned short)((o[u >> 1] >> (16 * (u & 1))) & 0xffffu));
            }
          }
        } else {  // kEpiAccF32
          if (rv) {
            float* dst = static_cast<float*>(p.out) + (int64_t)row * p.ldo + col0;
            if (col0 + 32 <= p.N && ((p.ldo & 3) == 0)) {
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                float4 a = make_float4(__uint_as_float(v[4 * u]), __uint_as_float(v[4 * u + 1]),
                                       __uint_as_float(v[4 * u + 2]), __uint_as_float(v[4 * u + 3]));
                if (p.beta) {
                  const float4 o = reinterpret_cast<const float4*>(dst)[u];
                  a.x += o.x; a.y += o.y; a.z += o.z; a.w += o.w;
                }
                reinterpret_cast<float4*>(dst)[u] = a;
              }
            } else {
#pragma unroll
              for (int u = 0; u < 32; ++u)
                if (col0 + u < p.N) dst[u] = __uint_as_float(v[u]) + (p.beta ? dst[u] : 0.f);
            }
          }
        }
      }
      if constexpr (EPI == kEpiLsePartial) {
        if (rv) p.part[(int64_t)(2 * tn + half) * p.M + row] = make_float2(m_run, s_run);
      }
      // accumulator buffer b read: release it to the leader's MMA warp
      tc_fence_before();
      __syncwarp();
      if (lane == 0) arrive_leader(&acc_empty[b]);
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // the peer's shared memory / TMEM stay alive until the pair's last MMA and arrival
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult qr;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}

// row-major bf16 [rows, cols] with row stride ld (elements), as a 3-D map {cols, 1, rows} with a
// {64, 1, box_rows} SWIZZLE_128B box (64 bf16 = one 128-byte swizzle row)
tt_status make_map(CUtensorMap* m, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
  auto fn = encoder();
  if (!fn) { set_error("cuTensorMapEncodeTiled unavailable"); return TT_ERR_CUDA; }
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) || (ld * 2) % 16) {
    set_error("gemm operand: 16-byte aligned base and row stride required");
    return TT_ERR_ALIGNMENT;
  }
  cuuint64_t dims[3] = {(cuuint64_t)cols, 1, (cuuint64_t)rows};
  cuuint64_t strides[2] = {(cuuint64_t)ld * 2, (cuuint64_t)ld * 2};
  cuuint32_t box[3] = {64, 1, (cuuint32_t)box_rows};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { set_error("cuTensorMapEncodeTiled failed (%d)", (int)r); return TT_ERR_CUDA; }
  return TT_OK;
}

template <int EPI>
tt_status launch(const CUtensorMap& ma, const CUtensorMap& mb, const Args& a, cudaStream_t st) {
  auto kern = gemm_pair_kernel<EPI>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
  if (e != cudaSuccess) { set_error("gemm: smem attribute: %s", cudaGetErrorString(e)); return TT_ERR_CUDA; }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int n_tiles = a.tiles_m * a.tiles_n;
  const int pairs = std::max(1, std::min(sms / 2, n_tiles));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(2 * pairs));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, ma, mb, a);
  if (e != cudaSuccess) { set_error("gemm_pair_kernel launch: %s", cudaGetErrorString(e)); return TT_ERR_CUDA; }
  count_launch();
  return check_launch("gemm_pair_kernel");
}

}  // namespace

// D[M, N] = A . B with A stored row-major [M, K] (a_mn = 0) or [K, M] (a_mn = 1), B stored row-major
// [N, K] (b_mn = 0) or [K, N] (b_mn = 1); lda / ldb are the stored row strides (elements).
tt_status gemm_run(int epi, int M, int N, int K, const void* A, int64_t lda, int a_mn, const void* B, int64_t ldb,
                   int b_mn, const GemmEpilogue& ep, cudaStream_t st) {
  if (M <= 0 || N <= 0 || K <= 0) return TT_OK;
  CUtensorMap ma, mb;
  tt_status s;
  if ((s = a_mn ? make_map(&ma, A, K, M, lda, 64) : make_map(&ma, A, M, K, lda, 128))) return s;
  if ((s = b_mn ? make_map(&mb, B, K, N, ldb, 64) : make_map(&mb, B, N, K, ldb, 128))) return s;
  Args a{};
  a.M = M; a.N = N; a.K = K;
  a.a_mn = a_mn; a.b_mn = b_mn;
  a.tiles_m = (M + 255) / 256;
  a.tiles_n = (N + 255) / 256;
  a.out = ep.out; a.ldo = ep.ldo; a.beta = ep.beta;
  a.col_offset = ep.col_offset; a.vocab = ep.vocab; a.part = reinterpret_cast<float2*>(ep.part);
  a.max_t = ep.max_t; a.tgt_cnt = ep.tgt_cnt; a.tgt_y = ep.tgt_y; a.tgt_w = ep.tgt_w; a.tgt_x = ep.tgt_x;
  a.lse2 = ep.lse2; a.g_omega = ep.g_omega; a.gamma = ep.gamma;
  a.wait_mode = 0;
  if (const char* w = dev_getenv("TT_GEMM_WAIT")) a.wait_mode = atoi(w);
  switch (epi) {
    case kEpiStoreBF16: return launch<kEpiStoreBF16>(ma, mb, a, st);
    case kEpiAccF32: return launch<kEpiAccF32>(ma, mb, a, st);
    case kEpiLsePartial: return launch<kEpiLsePartial>(ma, mb, a, st);
    case kEpiDlogits: return launch<kEpiDlogits>(ma, mb, a, st);
    default: set_error("gemm: bad epilogue %d", epi); return TT_ERR_INVALID_ARGUMENT;
  }
}

}  // namespace gemm
}  // namespace tt
