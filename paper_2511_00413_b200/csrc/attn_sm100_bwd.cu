// attn_sm100_bwd.cu — tree-masked attention backward with Gradient Restoration on sm_100a
// (tcgen05 + TMEM + TMA).
//
// What it computes (Eqs. 2, 14-16, 20-21, P:130-135 / P:408-436 / P:483-497; readings R6, R12):
//   omega_i = w_i (restore) or 1,  P_ij = exp(scale q_i.k_j - LSE_i),  D_i = dO_i.O_i
//   dV_j  = sum_i omega_i P_ij dO_i
//   dS_ij = omega_i P_ij (dO_i.v_j - D_i)
//   dK_j  = scale sum_i dS_ij q_i,   dQ_i = scale sum_j dS_ij k_j      over j <= i < E_j
// The tree-scale enters as a per-query-column factor on P and dS in registers:
// dO and D stay unscaled and no restored copy of dO is ever materialised.
//
// Design — key-stationary: one CTA owns a 128-key block kb of one kv head and
// walks the contiguous query range [128 kb, maxE_kb) (exact: the queries that see key j are
// [j, E_j)) in 64-row query tiles, for every q head of the GQA group.  K and V stay in shared
// memory; dK and dV accumulate in TMEM across all iterations.
//   warp 0     producer: TMA of K, V once; per iteration TMA of Q_i, dO_i (64 x 128) into a
//              3-stage ring, plus LSE (log2), D and w of the 64 rows staged by the 32 lanes
//   warp 1     TMEM allocator + MMA issuer (one thread).  Per iteration:
//                S^T = K Q^T, dP^T = V dO^T            (M=128 keys, N=64 queries, K=d)
//                dV += P^T dO      (A = P^T from TMEM)  (M=128, N=128, K=64)
//                dK += dS^T Q      (A = dS^T from smem) (M=128, N=128, K=64)
//                dQ^T = K^T dS^T   (A = K^T MN-major)   (M=128 (d), N=64, K=128)
//              S^T / dP^T are double buffered so the next tile's products overlap this tile's
//              element-wise work; dQ^T reuses the dP^T buffer once the softmax has read it.
//   warps 2-5  element-wise: one thread per key row (TMEM lane); P^T, dS^T with the tree-scale,
//              P^T -> TMEM (bf16), dS^T -> smem (bf16, SWIZZLE_128B); final dK/dV epilogue
//   warps 6-9  dQ drain: one thread per head-dim lane of dQ^T; coalesced fp32 reductions into the
//              fp32 dQ accumulator (128 contiguous bytes per warp instruction)
// TMEM columns: dV 0-127 | dK 128-255 | S^T[2] 256-383 | dP^T[2] (or dQ^T) 384-511.
#include <cudaTypedefs.h>

#include "sm100_ptx.cuh"
#include "tt_internal.cuh"

namespace tt {
namespace {
using namespace sm100;

constexpr int kD = 128;
constexpr int kBQ = 64;
constexpr int kQStages = 3;
constexpr int kBwdThreads = 320;
constexpr uint32_t kKVTile = 128 * kD * 2;     // 32 KB (two 16 KB chunks of 128 rows x 128 B)
constexpr uint32_t kKVChunk = 128 * 64 * 2;    // 16 KB
constexpr uint32_t kQTile = kBQ * kD * 2;      // 16 KB (two 8 KB chunks of 64 rows x 128 B)
constexpr uint32_t kQChunk = kBQ * 64 * 2;     // 8 KB
constexpr uint32_t kOffK = 0;
constexpr uint32_t kOffV = kKVTile;
constexpr uint32_t kOffQS = 2 * kKVTile;                     // stage s: Q at +s*32K, dO at +s*32K+16K
constexpr uint32_t kOffStats = kOffQS + kQStages * 2 * kQTile;  // stage s: lse | D | w (256 B each)
constexpr uint32_t kOffDS = ((kOffStats + kQStages * 1024 + 1023) / 1024) * 1024;  // dS^T[2], 16 KB each
constexpr uint32_t kDSTile = 128 * kBQ * 2;
constexpr uint32_t kOffBar = kOffDS + 2 * kDSTile;
constexpr uint32_t kNumBars = 1 + 2 * kQStages + 8 + 1;
constexpr uint32_t kOffMisc = kOffBar + kNumBars * 8;
constexpr uint32_t kSmemBytes = kOffMisc + 16 + 1024;

constexpr uint32_t kColDV = 0, kColDK = 128, kColS = 256, kColP = 384;

struct BwdParams {
  int64_t N;
  int hq, hkv, g, nb;
  int restore;
  float scale, scale_log2;
  const int32_t* E;
  const int32_t* kmaxE;
  const int32_t* w;
  const float* lse;
  const float* Dvec;
  float* dq_acc;
  __nv_bfloat16* dk;
  __nv_bfloat16* dv;
};

__global__ void __launch_bounds__(kBwdThreads, 1)
    tree_attn_bwd_sm100(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                        const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmdO,
                        const BwdParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar);
  uint64_t* kv_full = bars;
  uint64_t* q_full = bars + 1;
  uint64_t* q_empty = q_full + kQStages;
  uint64_t* s_full = q_empty + kQStages;  // [2]
  uint64_t* sm_done = s_full + 2;         // [2]
  uint64_t* dq_full = sm_done + 2;        // [2]
  uint64_t* dq_free = dq_full + 2;        // [2]
  uint64_t* acc_done = dq_free + 2;
  uint32_t* misc = reinterpret_cast<uint32_t*>(smem + kOffMisc);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kb = (int)(blockIdx.x / p.hkv);
  const int hk = (int)(blockIdx.x % p.hkv);
  const int64_t k0 = (int64_t)kb * 128;
  const int qt0 = (int)(k0 / kBQ);                                    // first 64-row query tile
  const int qt1 = (int)((p.kmaxE[kb] + kBQ - 1) / kBQ);                // exclusive
  const int nq = qt1 - qt0;
  const int n_it = nq * p.g;                                          // (head, query tile) pairs

  if (warp == 1) {
    if (lane == 0) {
      mbar_init(kv_full, 1);
      for (int s = 0; s < kQStages; ++s) { mbar_init(&q_full[s], 33); mbar_init(&q_empty[s], 1); }
      for (int b = 0; b < 2; ++b) {
        mbar_init(&s_full[b], 1);
        mbar_init(&sm_done[b], 128);
        mbar_init(&dq_full[b], 1);
        mbar_init(&dq_free[b], 128);
      }
      mbar_init(acc_done, 1);
      mbar_fence_init();
    }
    __syncwarp();
    tmem_alloc(&misc[0], 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = misc[0];

  if (warp == 0) {
    // ===================== producer warp =====================
    // lane 0 issues the TMA tiles; all 32 lanes stage LSE (as log2), D and w for the 64 query rows
    // with plain loads (the [hq, N] rows are not 16-byte aligned for ragged N) and arrive.
    if (lane == 0) {
      tma_prefetch(&tmQ);
      tma_prefetch(&tmK);
      tma_prefetch(&tmV);
      tma_prefetch(&tmdO);
      mbar_expect_tx(kv_full, 2 * kKVTile);
      for (int c = 0; c < 2; ++c) {
        tma_load_3d(smem + kOffK + c * kKVChunk, &tmK, kv_full, c * 64, hk, (int)k0);
        tma_load_3d(smem + kOffV + c * kKVChunk, &tmV, kv_full, c * 64, hk, (int)k0);
      }
    }
    for (int it = 0; it < n_it; ++it) {
      const int s = it % kQStages;
      if (it >= kQStages) mbar_wait(&q_empty[s], ((it / kQStages) - 1) & 1);
      const int h = hk * p.g + it / nq;
      const int q0 = (qt0 + it % nq) * kBQ;
      if (lane == 0) {
        uint8_t* qd = smem + kOffQS + s * 2 * kQTile;
        mbar_expect_tx(&q_full[s], 2 * kQTile);
        for (int c = 0; c < 2; ++c) {
          tma_load_3d(qd + c * kQChunk, &tmQ, &q_full[s], c * 64, h, q0);
          tma_load_3d(qd + kQTile + c * kQChunk, &tmdO, &q_full[s], c * 64, h, q0);
        }
      }
      float* st = reinterpret_cast<float*>(smem + kOffStats + s * 1024);
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int c = lane + 32 * u;
        const int64_t i = (int64_t)q0 + c;
        const bool in = i < p.N;
        st[c] = in ? p.lse[(int64_t)h * p.N + i] * kLog2e : 0.f;
        st[64 + c] = in ? p.Dvec[(int64_t)h * p.N + i] : 0.f;
        st[128 + c] = (in && p.restore) ? (float)p.w[i] : 1.f;
      }
      mbar_arrive(&q_full[s]);
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ===================== MMA issuer =====================
      constexpr uint32_t idSP = idesc_bf16(128, kBQ, 0, 0);   // K/V (K-major) x Q/dO^T (K-major)
      constexpr uint32_t idVK = idesc_bf16(128, 128, 0, 1);   // P^T/dS^T (K-major) x dO/Q (MN-major)
      constexpr uint32_t idQ = idesc_bf16(128, kBQ, 1, 1);    // K^T (MN-major) x dS^T (MN-major)
      const uint32_t kb_s = smem_u32(smem + kOffK), vb_s = smem_u32(smem + kOffV);
      auto issue_SP = [&](int it) {
        const int s = it % kQStages, b = it & 1;
        const uint32_t qb = smem_u32(smem + kOffQS + s * 2 * kQTile);
        const uint32_t ob = qb + kQTile;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t offk = (kk >> 2) * kKVChunk + (kk & 3) * 32;
          const uint32_t offq = (kk >> 2) * kQChunk + (kk & 3) * 32;
          mma_ss(tmem + kColS + 64 * b, sdesc(kb_s + offk, 16, 1024), sdesc(qb + offq, 16, 1024), idSP, kk > 0);
        }
        return ob;
      };
      auto issue_dP = [&](int it) {
        const int s = it % kQStages, b = it & 1;
        const uint32_t ob = smem_u32(smem + kOffQS + s * 2 * kQTile) + kQTile;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t offk = (kk >> 2) * kKVChunk + (kk & 3) * 32;
          const uint32_t offq = (kk >> 2) * kQChunk + (kk & 3) * 32;
          mma_ss(tmem + kColP + 64 * b, sdesc(vb_s + offk, 16, 1024), sdesc(ob + offq, 16, 1024), idSP, kk > 0);
        }
      };
      mbar_wait(kv_full, 0);
      for (int it = 0; it < n_it && it < 2; ++it) {
        mbar_wait(&q_full[it % kQStages], (it / kQStages) & 1);
        tc_fence_after();
        issue_SP(it);
        issue_dP(it);
        mma_commit(&s_full[it & 1]);
      }
      for (int it = 0; it < n_it; ++it) {
        const int s = it % kQStages, b = it & 1;
        const uint32_t qb = smem_u32(smem + kOffQS + s * 2 * kQTile);
        const uint32_t ob = qb + kQTile;
        const uint32_t dsb = smem_u32(smem + kOffDS + b * kDSTile);
        mbar_wait(&sm_done[b], (it >> 1) & 1);
        tc_fence_after();
        // dV += P^T dO   (A: P^T bf16 in TMEM over S^T[b]; B: dO MN-major, LBO = 8 KB d-chunk)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_ts(tmem + kColDV, tmem + kColS + 64 * b + kk * 8, sdesc(ob + kk * 2048, kQChunk, 1024), idVK,
                 (it > 0 || kk > 0) ? 1u : 0u);
        // dK += dS^T Q   (A: dS^T K-major 128 x 64 in smem; B: Q MN-major)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_ss(tmem + kColDK, sdesc(dsb + kk * 32, 16, 1024), sdesc(qb + kk * 2048, kQChunk, 1024), idVK,
                 (it > 0 || kk > 0) ? 1u : 0u);
        // dQ^T = K^T dS^T   (A: K MN-major, LBO = 16 KB d-chunk; B: dS^T MN-major, one 64-wide group)
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_ss(tmem + kColP + 64 * b, sdesc(kb_s + kk * 2048, kKVChunk, 1024), sdesc(dsb + kk * 2048, kDSTile, 1024),
                 idQ, kk > 0);
        mma_commit(&dq_full[b]);
        mma_commit(&q_empty[s]);
        if (it + 2 < n_it) {
          mbar_wait(&q_full[(it + 2) % kQStages], ((it + 2) / kQStages) & 1);
          tc_fence_after();
          issue_SP(it + 2);
          mbar_wait(&dq_free[b], (it >> 1) & 1);
          tc_fence_after();
          issue_dP(it + 2);
          mma_commit(&s_full[b]);
        }
      }
      mma_commit(acc_done);
    }
  } else if (warp < 6) {
    // ===================== element-wise (one thread per key row) =====================
    const int q4 = warp & 3;
    const int r = q4 * 32 + lane;
    const int64_t j = k0 + r;
    const uint32_t tl = tmem + ((uint32_t)(q4 * 32) << 16);
    const int Ej = (j < p.N) ? p.E[j] : -1;
    const float sl2 = p.scale_log2;
    for (int it = 0; it < n_it; ++it) {
      const int s = it % kQStages, b = it & 1;
      const int q0 = (qt0 + it % nq) * kBQ;
      mbar_wait(&s_full[b], (it >> 1) & 1);
      tc_fence_after();
      const float4* st_lse = reinterpret_cast<const float4*>(smem + kOffStats + s * 1024);
      const float4* st_D = reinterpret_cast<const float4*>(smem + kOffStats + s * 1024 + 256);
      const float4* st_w = reinterpret_cast<const float4*>(smem + kOffStats + s * 1024 + 512);
      // rows of this key that need no mask: j <= q0 and q0 + 63 < min(E_j, N)
      const bool nomask = __all_sync(0xffffffffu, (j <= q0) && ((int64_t)q0 + kBQ - 1 < (int64_t)Ej) &&
                                                      ((int64_t)q0 + kBQ - 1 < p.N));
      uint8_t* drow = smem + kOffDS + b * kDSTile + r * 128;
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {  // two halves of 32 query columns (keeps registers < 168)
        uint32_t sv[32], pv[32];
        tmem_ld32(tl + kColS + 64 * b + 32 * hh, sv);
        tmem_ld32(tl + kColP + 64 * b + 32 * hh, pv);
        tmem_wait_ld();
        uint32_t pwk[16], dsk[16];
#pragma unroll
        for (int c4 = 0; c4 < 8; ++c4) {
          const int cg = 8 * hh + c4;  // float4 group within the 64 columns
          const float4 L = st_lse[cg];
          const float4 Dd = st_D[cg];
          const float4 W = st_w[cg];
          const float Lv[4] = {L.x, L.y, L.z, L.w};
          const float Dv[4] = {Dd.x, Dd.y, Dd.z, Dd.w};
          const float Wv[4] = {W.x, W.y, W.z, W.w};
          float pw[4], ds[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int c = 4 * c4 + u;
            const int64_t i = q0 + 32 * hh + c;
            float pr = ex2(fmaf(__uint_as_float(sv[c]), sl2, -Lv[u]));
            if (!nomask) {
              const bool ok = (j <= i) && (i < (int64_t)Ej) && (i < p.N);
              pr = ok ? pr : 0.f;
            }
            pw[u] = Wv[u] * pr;
            ds[u] = pw[u] * (__uint_as_float(pv[c]) - Dv[u]);
          }
          pwk[2 * c4] = pack_bf16(pw[0], pw[1]);
          pwk[2 * c4 + 1] = pack_bf16(pw[2], pw[3]);
          dsk[2 * c4] = pack_bf16(ds[0], ds[1]);
          dsk[2 * c4 + 1] = pack_bf16(ds[2], ds[3]);
        }
        // P^T (bf16) over S^T[b] in TMEM: columns [16 hh, 16 hh + 16)
        tmem_st16(tl + kColS + 64 * b + 16 * hh, pwk);
        // dS^T row r (128 B) into the SWIZZLE_128B smem tile: 16-byte chunk c at (c ^ (r & 7))
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int ch = 4 * hh + c;
          *reinterpret_cast<uint4*>(drow + ((ch ^ (r & 7)) << 4)) =
              make_uint4(dsk[4 * c], dsk[4 * c + 1], dsk[4 * c + 2], dsk[4 * c + 3]);
        }
      }
      tmem_wait_st();
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&sm_done[b]);
    }
    // ---- epilogue: dV, dK (scaled) rows of this key -> bf16 ----
    mbar_wait(acc_done, 0);
    tc_fence_after();
#pragma unroll 1
    for (int which = 0; which < 2; ++which) {
      const uint32_t col = which == 0 ? kColDV : kColDK;
      const float mul = which == 0 ? 1.f : p.scale;
      __nv_bfloat16* dst = (which == 0 ? p.dv : p.dk) + (j * p.hkv + hk) * kD;
#pragma unroll 1
      for (int cc = 0; cc < 4; ++cc) {
        uint32_t ov[32];
        tmem_ld32(tl + col + 32 * cc, ov);
        tmem_wait_ld();
        if (j < p.N) {
          uint32_t pk[16];
#pragma unroll
          for (int u = 0; u < 16; ++u)
            pk[u] = pack_bf16(__uint_as_float(ov[2 * u]) * mul, __uint_as_float(ov[2 * u + 1]) * mul);
          uint4* d4 = reinterpret_cast<uint4*>(dst + 32 * cc);
#pragma unroll
          for (int u = 0; u < 4; ++u) d4[u] = make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
        }
      }
    }
  } else {
    // ===================== dQ drain (one thread per head-dim lane of dQ^T) =====================
    const int q4 = warp & 3;
    const int dl = q4 * 32 + lane;
    const uint32_t tl = tmem + ((uint32_t)(q4 * 32) << 16);
    for (int it = 0; it < n_it; ++it) {
      const int b = it & 1;
      const int h = hk * p.g + it / nq;
      const int q0 = (qt0 + it % nq) * kBQ;
      mbar_wait(&dq_full[b], (it >> 1) & 1);
      tc_fence_after();
      uint32_t v0[32], v1[32];
      tmem_ld32(tl + kColP + 64 * b, v0);
      tmem_ld32(tl + kColP + 64 * b + 32, v1);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(&dq_free[b]);
      const int nrow = (int)imin64(kBQ, p.N - q0);
      const int64_t rs = (int64_t)p.hq * kD;
      float* ptr = p.dq_acc + ((int64_t)q0 * p.hq + h) * kD + dl;
      if (nrow == kBQ) {
#pragma unroll
        for (int c = 0; c < 32; ++c) { atomicAdd(ptr, __uint_as_float(v0[c]) * p.scale); ptr += rs; }
#pragma unroll
        for (int c = 0; c < 32; ++c) { atomicAdd(ptr, __uint_as_float(v1[c]) * p.scale); ptr += rs; }
      } else {
#pragma unroll
        for (int c = 0; c < 32; ++c) { if (c < nrow) atomicAdd(ptr, __uint_as_float(v0[c]) * p.scale); ptr += rs; }
#pragma unroll
        for (int c = 0; c < 32; ++c) { if (32 + c < nrow) atomicAdd(ptr, __uint_as_float(v1[c]) * p.scale); ptr += rs; }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// dQ fp32 accumulator -> bf16 output
__global__ void __launch_bounds__(256) dq_convert_kernel(const float4* __restrict__ acc, uint2* __restrict__ out,
                                                         int64_t n4) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 a = acc[i];
    out[i] = make_uint2(pack_bf16(a.x, a.y), pack_bf16(a.z, a.w));
  }
}

}  // namespace

tt_status sm100_attn_bwd(const tt_packed& pk, const void* q, const void* k, const void* v, const float* lse,
                         const float* Dvec, const void* dout, int restore, int hq, int hkv, int d, float scale,
                         float* dq_acc, void* dq, void* dk, void* dv, cudaStream_t st) {
  if (d != kD) { set_error("sm100_attn_bwd: d must be 128"); return TT_ERR_UNSUPPORTED; }
  CUtensorMap mq, mk, mv, mdo;
  tt_status s;
  const auto BF = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  const auto SW = CU_TENSOR_MAP_SWIZZLE_128B;
  if ((s = make_tmap_thd(&mq, q, pk.n_tokens, hq, d, kBQ, BF, 2, SW, 64))) return s;
  if ((s = make_tmap_thd(&mdo, dout, pk.n_tokens, hq, d, kBQ, BF, 2, SW, 64))) return s;
  if ((s = make_tmap_thd(&mk, k, pk.n_tokens, hkv, d, 128, BF, 2, SW, 64))) return s;
  if ((s = make_tmap_thd(&mv, v, pk.n_tokens, hkv, d, 128, BF, 2, SW, 64))) return s;
  BwdParams prm;
  prm.N = pk.n_tokens;
  prm.hq = hq;
  prm.hkv = hkv;
  prm.g = hq / hkv;
  prm.nb = pk.n_blk;
  prm.restore = restore ? 1 : 0;
  prm.scale = scale;
  prm.scale_log2 = scale * kLog2e;
  prm.E = pk.E;
  prm.kmaxE = pk.kblk_maxE;
  prm.w = pk.w;
  prm.lse = lse;
  prm.Dvec = Dvec;
  prm.dq_acc = dq_acc;
  prm.dk = static_cast<__nv_bfloat16*>(dk);
  prm.dv = static_cast<__nv_bfloat16*>(dv);
  cudaError_t e = cudaFuncSetAttribute(tree_attn_bwd_sm100, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
  if (e != cudaSuccess) { set_error("sm100_attn_bwd: smem attribute: %s", cudaGetErrorString(e)); return TT_ERR_CUDA; }
  const unsigned grid = (unsigned)pk.n_blk * hkv;
  tree_attn_bwd_sm100<<<grid, kBwdThreads, kSmemBytes, st>>>(mq, mk, mv, mdo, prm);
  count_launch();
  if ((s = check_launch("tree_attn_bwd_sm100"))) return s;
  const int64_t n4 = pk.n_tokens * hq * d / 4;
  dq_convert_kernel<<<(unsigned)std::min<int64_t>((n4 + 255) / 256, 148 * 16), 256, 0, st>>>(
      reinterpret_cast<const float4*>(dq_acc), reinterpret_cast<uint2*>(dq), n4);
  count_launch();
  return check_launch("dq_convert_kernel");
}

}  // namespace tt
