// attn_sm100_bwd_flat.cu — the non-persistent tree-attention backward (one CTA per (key block, kv head),
// K / V written into TMEM by the drain warpgroup from global memory): the round-2-start kernel, kept for
// trees whose work items are long.  sm100_attn_bwd (attn_sm100_bwd.cu) dispatches here when the mean
// query tiles per item is at least kBwdFlatMinTilesPerItem (tt_internal.cuh): on those trees the persistent kernel gains
// nothing at its item boundaries and measured 1-2% slower per tile (profiles/r2q_bwd_ab.txt); on small
// trees (agentic8k) the persistent kernel is 8% faster.  Same workspace, preprocessing, dQ conversion
// and a6 partials as the persistent kernel (attn_sm100_bwd.cu).
//
// (the round-2-start kernel, unchanged apart from its name and this launcher:)
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
// [j, E_j)) in 64-row query tiles, for every q head of the GQA group.  K and V are resident in TMEM
// (K also in shared memory as dQ^T's A operand); dK and dV accumulate in TMEM across all iterations.
//   warp 0     producer: TMA of K once; per iteration TMA of Q_i, dO_i (64 x 128) into a 3-stage
//              ring, plus LSE (log2), D and w of the 64 rows (bulk copies)
//   warp 1     TMEM allocator + MMA issuer (one elected thread).  Per iteration:
//                S^T = K Q^T, dP^T = V dO^T   (TS: A = K / V from TMEM; M=128 keys, N=64 queries, K=d)
//                dV += P^T dO      (A = P^T from TMEM)  (M=128, N=128, K=64)
//                dK += dS^T Q      (A = dS^T from smem) (M=128, N=128, K=64)
//                dQ^T = K^T dS^T   (A = K^T MN-major)   (M=128 (d), N=64, K=128) into the dP^T columns
//              Issue order per tile i: [P^T(i) ready] dV(i), S(i+1); [dS^T(i) ready] dQ^T(i), dK(i);
//              [dQ^T(i) drained] dP(i+1).  S^T, dP^T / dQ^T single buffered (TMEM is full).
//              Bounds: N = 64 MMAs run at 45 (TS) / 53 (SS) cycles against a
//              32-cycle floor, and sustained the kernel runs at the board power cap, where the dQ L2
//              reduce and the element-wise math each cost ~14% of its energy.
//   warps 2-9  two warpgroups sharing the 4 TMEM lane quadrants; warpgroup wg owns query columns
//              [32 wg, 32 wg + 32) of each tile.  Element-wise (one thread per key row): P^T, dS^T
//              with the tree-scale, P^T -> TMEM (bf16), dS^T -> smem (bf16, SWIZZLE_128B).
//              Epilogue: warpgroup 0 writes dV, warpgroup 1 writes dK.
//   warps 10-13 dQ drain warpgroup (one thread per head-dim lane of dQ^T): copies K and V rows into
//              TMEM at the start; per tile it reads the 64 query columns of dQ^T from TMEM, releases
//              the columns to the MMA issuer, and adds them into the fp32 dQ accumulator through two
//              16 KB smem stages (32 query rows x 128 fp32 each, [row][dim]) with TMA bulk tensor
//              reductions (cp.reduce.async.bulk.tensor .add.f32).
// TMEM columns: dV 0-127 | dK 128-255 | S^T 256-319 | K 320-383 | dP^T / dQ^T 384-447 | V 448-511.
#include <cudaTypedefs.h>

#include <cstdlib>

#include "sm100_ptx.cuh"

// Development cycle counters (per-role wait / compute time, read back with tt_debug_*_counters):
// compiled in only with -DTT_PROFILE_COUNTERS; otherwise TT_CLK() is a constant and the bookkeeping
// folds away.
#ifdef TT_PROFILE_COUNTERS
#define TT_CLK() clock64()
#else
#define TT_CLK() 0ll
#endif
#include "tt_internal.cuh"

namespace tt {
namespace {
using namespace sm100;

constexpr int kD = 128;
constexpr int kBQ = 64;
constexpr int kQStages = 3;
// element-wise warpgroups: kNWG, each owning kCW query columns of every 64-row tile
#ifndef TT_BWD_NWG
#define TT_BWD_NWG 2  // measured: 4 warpgroups (16 columns each, 80 registers) within noise of 2 (profiles/r1f_bwd_nwg_ab.txt)
#endif
constexpr int kNWG = TT_BWD_NWG;
constexpr int kCW = 64 / kNWG;
static_assert(kNWG == 2 || kNWG == 4, "2 or 4 element-wise warpgroups");
constexpr int kDrainWarp0 = 2 + 4 * kNWG;                  // first warp of the dQ drain warpgroup
constexpr int kBwdThreads = 32 * (kDrainWarp0 + 4);        // producer, MMA, element-wise, drain
constexpr uint32_t kKVTile = 128 * kD * 2;     // 32 KB (two 16 KB chunks of 128 rows x 128 B)
constexpr uint32_t kKVChunk = 128 * 64 * 2;    // 16 KB
constexpr uint32_t kQTile = kBQ * kD * 2;      // 16 KB (two 8 KB chunks of 64 rows x 128 B)
constexpr uint32_t kQChunk = kBQ * 64 * 2;     // 8 KB
constexpr uint32_t kOffK = 0;
constexpr uint32_t kOffV = kKVTile;
constexpr uint32_t kOffQS = 2 * kKVTile;                     // stage s: Q at +s*32K, dO at +s*32K+16K
constexpr uint32_t kDSTile = 128 * kBQ * 2;
constexpr uint32_t kOffDS = kOffQS + kQStages * 2 * kQTile;      // dS^T[2], 16 KB each (1024-aligned)
constexpr uint32_t kOffDQ = kOffDS + 2 * kDSTile;                 // dQ staging: 2 stages x 32 rows x 128 fp32
constexpr uint32_t kDQStage = 32 * kD * 4;
constexpr uint32_t kStatBytes = 768;                              // per stage: -LSE2 | -D | w (256 B each)
constexpr uint32_t kOffStats = kOffDQ + 2 * kDQStage;
constexpr uint32_t kOffBar = kOffStats + kQStages * kStatBytes;
constexpr uint32_t kNumBars = 1 + 2 * kQStages + 12 + 1 + 1;
constexpr uint32_t kOffMisc = kOffBar + kNumBars * 8;
// The dynamic shared-memory window is 1024-byte aligned on sm_100 (checked at run time; the kernel
// traps otherwise), so no alignment slack is reserved.
constexpr uint32_t kOffRed = kOffMisc + 16;                       // a6 reduction scratch: double [kNWG][4]
// (no static __shared__ in this kernel: it would shift the 1024-byte aligned dynamic window)
constexpr uint32_t kSmemBytes = kOffRed + 32 * kNWG;
static_assert(kSmemBytes <= 232448, "backward kernel exceeds 227 KB of shared memory");

// TT_BWD_KTMEM: K resident in TMEM (A operand of S^T = K Q^T as a TS MMA: the 32 KB per tile of K
// re-reads from shared memory disappear) at the price of a single S^T buffer.
#ifndef TT_BWD_KTMEM
#define TT_BWD_KTMEM 1
#endif
constexpr bool kKT = TT_BWD_KTMEM != 0;
// TT_BWD_VTMEM (requires KTMEM): V resident in TMEM too (dP^T = V dO^T as a TS MMA: the 32 KB per tile
// of V reads from shared memory disappear) and dQ^T accumulates in the dP^T columns once the element-wise
// warps have read dP^T; dP^T(i+1) is issued after the drain has read dQ^T(i).
#ifndef TT_BWD_VTMEM
#define TT_BWD_VTMEM 1
#endif
constexpr bool kVT = kKT && TT_BWD_VTMEM != 0;
// TMEM columns: dV 0-127 | dK 128-255 | S^T 256-319 (KTMEM) or S^T x2 256-383 | K 320-383 (KTMEM) |
// dP^T 384-447 (VTMEM: dP^T, then dQ^T) | dQ^T 448-511 (VTMEM: V)
constexpr uint32_t kColDV = 0, kColDK = 128, kColS = 256, kColK = 320, kColP = 384;
constexpr uint32_t kColQ = kVT ? kColP : 448, kColV = 448;

// development instrumentation (TT_DEBUG_BWD & 8): per-role cycle counters summed over CTAs
__device__ unsigned long long g_bwd_dbg[16];  // (dev counters: not read back for the flat kernel)

struct BwdParams {
  int64_t N;
  int hq, hkv, g, nb;
  int restore;
  int chunk;  // CTA order: key blocks in chunks of `chunk`; within a chunk the kv heads outermost (1 = heads
              // fastest, >= nb = head-major: the Q / dO / dQ rows of one head group stay L2-resident)
  int wait;  // dev A/B (TT_WAIT_HINT): suspend-hint waits, bit 0 producer, 1 consumers, 2 epilogue
  int order;   // dev A/B (TT_BWD_ORDER): bit 0 issues dP(i+1) before dK(i)
  int l2hint;  // dev A/B (TT_BWD_L2HINT): bit 0/1 dQ reduce evict_last / evict_first, bit 2/3 Q / dO loads evict_last / evict_first
  int walk;  // query-tile walk (TT_BWD_WALK, dev A/B): bit 0 descending from maxE, bit 1 heads inner
  int dbg;  // development ablations (TT_DEBUG_BWD): 1 skip dQ reduce, 2 reuse Q/dO stage (no reload), 4 skip elementwise math, 32 stage dQ but skip the L2 reduce
  float scale, scale_log2;
  const int32_t* E;
  const int32_t* kmaxE;
  int64_t Np;          // token dimension of the padded preprocess arrays (multiple of 128)
  const float* L2p;    // [hq][Np] LSE in log2 units
  const float* Dp;     // [hq][Np] D = dO . O
  const float* wf;     // [Np] tree-scale (or 1) as fp32
  float* dq_acc;
  __nv_bfloat16* dk;
  __nv_bfloat16* dv;
  double* part_kv;  // nullable: [grid][2] fp64 partial sums of squares of this CTA's dV (0) / dK (1) rows
  const __nv_bfloat16* kmat;  // K [N, hkv, 128] (KTMEM: rows copied into TMEM by the drain warpgroup)
  const __nv_bfloat16* vmat;  // V [N, hkv, 128] (VTMEM: likewise)
};

// work item `it` of a CTA -> (q head, first query row of the 64-row tile).  The shipped walk (GQA heads
// outer, query tiles ascending) advances a (tile, head) counter pair: no integer division per tile.
struct Walk {
  int qi = 0, hi = 0;
};
__device__ __forceinline__ void bwd_item(const BwdParams& p, int it, Walk& wk, int nq, int qt0, int hk, int& h, int& q0) {
  const int w = dev_dbg(p.walk);
  int qi = wk.qi, hi = wk.hi;
  if (w) {
    qi = (w & 2) ? it / p.g : it % nq;
    hi = (w & 2) ? it % p.g : it / nq;
  }
  if (++wk.qi == nq) { wk.qi = 0; ++wk.hi; }
  h = hk * p.g + hi;
  q0 = ((w & 1) ? (qt0 + nq - 1 - qi) : (qt0 + qi)) * kBQ;
}

// FOLD: the tree-scale is folded into the preprocessed LSE (L2p = -LSE log2e + log2 w, valid for w >= 0:
// integer trajectory counts, non-negative real weights, or restore off), so P w = exp2(s scale log2e + L2p)
// costs no multiply and no per-tile load of w; real-valued weights with some w < 0 take the multiply.
template <bool FOLD>
__global__ void __maxnreg__(kNWG == 4 ? 80 : 128)  // 22 warps: 6 per SMSP x 80 regs x 32 fit its 16K registers
    tree_attn_bwd_flat_sm100(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                        const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmdO,
                        const __grid_constant__ CUtensorMap tmdQ, const BwdParams p) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned base; pointer arithmetic on smem_raw keeps the shared address space visible to
  // the compiler (LDS/STS instead of generic LD/ST)
  uint8_t* smem = smem_raw;
  if (smem_u32(smem_raw) & 1023u) __trap();
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar);
  uint64_t* kv_full = bars;
  uint64_t* q_full = bars + 1;
  uint64_t* q_empty = q_full + kQStages;
  uint64_t* s_full = q_empty + kQStages;  // [2] S^T(i) in TMEM
  uint64_t* p_ready = s_full + 2;         // [2] P^T(i) packed back into S^T[b] (256 arrivals)
  uint64_t* ds_ready = p_ready + 2;       // [2] dS^T(i) in smem (256 arrivals)
  uint64_t* dq_full = ds_ready + 2;       // [2]
  uint64_t* dq_free = dq_full + 2;        // [2]
  uint64_t* dp_full = dq_free + 2;        // dP^T(i) in TMEM
  uint64_t* dp_free = dp_full + 1;        // dP^T(i) read by the element-wise warps (256 arrivals)
  uint64_t* acc_done = dp_free + 1;
  uint64_t* k_tmem = acc_done + 1;        // K written into TMEM (128 arrivals, KTMEM)
  uint32_t* misc = reinterpret_cast<uint32_t*>(smem + kOffMisc);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long t_kernel0 = TT_CLK();
  int kb, hk;
  {
    const int per = p.chunk * p.hkv, x = (int)blockIdx.x;
    const int ch = x / per, w = x - ch * per;
    const int len = min(p.chunk, p.nb - ch * p.chunk);
    hk = w / len;
    kb = ch * p.chunk + (w - hk * len);
  }
  const int64_t k0 = (int64_t)kb * 128;
  const int qt0 = (int)(k0 / kBQ);                                    // first 64-row query tile
  const int qt1 = (int)((p.kmaxE[kb] + kBQ - 1) / kBQ);                // exclusive
  const int nq = qt1 - qt0;
  const int n_it = nq * p.g;                                          // (head, query tile) pairs

  if (warp == 1) {
    if (lane == 0) {
      mbar_init(kv_full, 1);
      for (int s = 0; s < kQStages; ++s) { mbar_init(&q_full[s], 1); mbar_init(&q_empty[s], 1); }
      for (int b = 0; b < 2; ++b) {
        mbar_init(&s_full[b], 1);
        mbar_init(&p_ready[b], 128 * kNWG);
        mbar_init(&ds_ready[b], 128 * kNWG);
        mbar_init(&dq_full[b], 1);
        mbar_init(&dq_free[b], 128);
      }
      mbar_init(dp_full, 1);
      mbar_init(dp_free, 128 * kNWG);
      mbar_init(acc_done, 1);
      mbar_init(k_tmem, 128);
      mbar_fence_init();
    }
  }
  // barriers visible to all; the producer (warp 0, which never touches TMEM) starts its loads now,
  // while warp 1 allocates TMEM for the other warps (named barrier 5 over warps 1..)
  __syncthreads();
  uint32_t tmem = 0;
  if (warp != 0) {
    if (warp == 1) {
      tmem_alloc(&misc[0], 512);
      tmem_relinquish();
    }
    tc_fence_before();
    named_bar_sync(5, kBwdThreads - 32);
    tc_fence_after();
    tmem = misc[0];
  }

  if (warp == 0) {
    // ===================== producer (lane 0) =====================
    if (lane == 0) {
      tma_prefetch(&tmQ);
      tma_prefetch(&tmK);
      tma_prefetch(&tmV);
      tma_prefetch(&tmdO);
      mbar_expect_tx(kv_full, (kVT ? 1 : 2) * kKVTile);
      for (int c = 0; c < 2; ++c) {
        tma_load_3d(smem + kOffK + c * kKVChunk, &tmK, kv_full, c * 64, hk, (int)k0);
        if (!kVT) tma_load_3d(smem + kOffV + c * kKVChunk, &tmV, kv_full, c * 64, hk, (int)k0);
      }
    }
    if (lane == 0) {
      Walk wk;
      for (int it = 0; it < n_it; ++it) {
        const int s = it % kQStages;
        if (it >= kQStages) mbar_wait_role(&q_empty[s], ((it / kQStages) - 1) & 1, dev_dbg(p.wait) & 1);
        int h, q0;
        bwd_item(p, it, wk, nq, qt0, hk, h, q0);
        uint8_t* qd = smem + kOffQS + s * 2 * kQTile;
        uint8_t* st = smem + kOffStats + s * kStatBytes;
        if ((dev_dbg(p.dbg) & 2) && it >= kQStages) {
          mbar_arrive(&q_full[s]);
          continue;
        }
        mbar_expect_tx(&q_full[s], 2 * kQTile + 3 * 256);
        if (dev_dbg(p.l2hint) & 12) {
          const uint64_t pol = (dev_dbg(p.l2hint) & 4) ? policy_evict_last() : policy_evict_first();
          for (int c = 0; c < 2; ++c) {
            tma_load_3d_hint(qd + c * kQChunk, &tmQ, &q_full[s], c * 64, h, q0, pol);
            tma_load_3d_hint(qd + kQTile + c * kQChunk, &tmdO, &q_full[s], c * 64, h, q0, pol);
          }
        } else {
          for (int c = 0; c < 2; ++c) {
            tma_load_3d(qd + c * kQChunk, &tmQ, &q_full[s], c * 64, h, q0);
            tma_load_3d(qd + kQTile + c * kQChunk, &tmdO, &q_full[s], c * 64, h, q0);
          }
        }
        bulk_load_1d(st, p.L2p + (int64_t)h * p.Np + q0, 256, &q_full[s]);
        bulk_load_1d(st + 256, p.Dp + (int64_t)h * p.Np + q0, 256, &q_full[s]);
        bulk_load_1d(st + 512, p.wf + q0, 256, &q_full[s]);
      }
    }
  } else if (warp == 1) {
    {
      // ===================== MMA issuer (whole warp, one elected lane issues) =====================
      constexpr uint32_t idSP = idesc_bf16(128, kBQ, 0, 0);   // K/V (K-major) x Q/dO^T (K-major)
      constexpr uint32_t idVK = idesc_bf16(128, 128, 0, 1);   // P^T/dS^T (K-major) x dO/Q (MN-major)
      constexpr uint32_t idQ = idesc_bf16(128, kBQ, 1, 1);    // K^T (MN-major) x dS^T (MN-major)
      const uint32_t kb_s = warp_uniform(smem_u32(smem + kOffK)), vb_s = kb_s + kOffV;
      const uint32_t tm = warp_uniform(tmem);
      const uint32_t qs0 = kb_s + kOffQS, ds0 = kb_s + kOffDS;
      auto issue_SP = [&](int it) {
        const int s = it % kQStages, b = it & 1;
        const uint32_t qb = qs0 + s * 2 * kQTile;
        const uint32_t ob = qb + kQTile;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t offk = (kk >> 2) * kKVChunk + (kk & 3) * 32;
          const uint32_t offq = (kk >> 2) * kQChunk + (kk & 3) * 32;
          if constexpr (kKT)
            mma_ts_w(tm + kColS, tm + kColK + 8 * kk, sdesc(qb + offq, 16, 1024), idSP, kk > 0);
          else
            mma_ss_w(tm + kColS + 64 * b, sdesc(kb_s + offk, 16, 1024), sdesc(qb + offq, 16, 1024), idSP, kk > 0);
        }
        return ob;
      };
      auto issue_dP = [&](int it) {
        const int s = it % kQStages;
        const uint32_t ob = qs0 + s * 2 * kQTile + kQTile;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t offk = (kk >> 2) * kKVChunk + (kk & 3) * 32;
          const uint32_t offq = (kk >> 2) * kQChunk + (kk & 3) * 32;
          if constexpr (kVT)
            mma_ts_w(tm + kColP, tm + kColV + 8 * kk, sdesc(ob + offq, 16, 1024), idSP, kk > 0);
          else
            mma_ss_w(tm + kColP, sdesc(vb_s + offk, 16, 1024), sdesc(ob + offq, 16, 1024), idSP, kk > 0);
        }
      };
      // dQ^T = K^T dS^T   (A: K MN-major, LBO = 16 KB d-chunk; B: dS^T MN-major, one 64-wide group)
      auto issue_dQ = [&](uint32_t dsb) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_ss_w(tm + kColQ, sdesc(kb_s + kk * 2048, kKVChunk, 1024), sdesc(dsb + kk * 2048, kDSTile, 1024),
                   idQ, kk > 0);
      };
      // dK += dS^T Q   (A: dS^T K-major 128 x 64 in smem; B: Q MN-major)
      auto issue_dK = [&](uint32_t dsb, uint32_t qb, int it) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_ss_w(tm + kColDK, sdesc(dsb + kk * 32, 16, 1024), sdesc(qb + kk * 2048, kQChunk, 1024), idVK,
                   (it > 0 || kk > 0) ? 1u : 0u);
      };
      long long w_sm = 0, w_dq = 0, w_q = 0, t_start = TT_CLK();
      mbar_wait(kv_full, 0);
      // prologue: S(0) -> s_full[0], dP(0) -> dp_full, S(1) -> s_full[1]
      mbar_wait(&q_full[0], 0);
      if constexpr (kKT) mbar_wait(k_tmem, 0);
      tc_fence_after();
      issue_SP(0);
      mma_commit_w(&s_full[0]);
      issue_dP(0);
      mma_commit_w(dp_full);
      if (!kKT && n_it > 1) {
        mbar_wait(&q_full[1], 0);
        tc_fence_after();
        issue_SP(1);
        mma_commit_w(&s_full[1]);
      }
      // Per tile i the element-wise warps run two phases: P (needs S^T(i) only) then dS (needs
      // dP^T(i)).  Each product is issued as soon as its operand is ready, so the tensor pipe works
      // on tile i's dV / dK / dQ and tile i+1's dP / tile i+2's S while the warps run phase P of the
      // next tile, and the warps never wait for a product issued after their previous tile finished.
      for (int it = 0; it < n_it; ++it) {
        const int s = it % kQStages, b = it & 1;
        const uint32_t qb = qs0 + s * 2 * kQTile;
        const uint32_t ob = qb + kQTile;
        const uint32_t dsb = ds0 + b * kDSTile;
        const int pb = kKT ? 0 : b;
        { long long t0 = TT_CLK(); mbar_wait(&p_ready[pb], kKT ? (it & 1) : ((it >> 1) & 1)); w_sm += TT_CLK() - t0; }
        tc_fence_after();
        // dV += P^T dO   (A: P^T bf16 in TMEM over S^T[b]; B: dO MN-major, LBO = 8 KB d-chunk)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)  // P^T of query columns 16 kk.. : warpgroup 16 kk / kCW packed it at its own S^T columns
          mma_ts_w(tm + kColDV, tm + kColS + 64 * pb + kCW * ((16 * kk) / kCW) + 8 * (((16 * kk) % kCW) / 16),
                   sdesc(ob + kk * 2048, kQChunk, 1024),
                   idVK, (it > 0 || kk > 0) ? 1u : 0u);
        // KTMEM: the single S^T buffer takes S^T(it+1) right after dV(it) has read P^T(it) from it
        if (kKT && it + 1 < n_it) {
          { long long t0 = TT_CLK(); mbar_wait(&q_full[(it + 1) % kQStages], ((it + 1) / kQStages) & 1); w_q += TT_CLK() - t0; }
          tc_fence_after();
          issue_SP(it + 1);
          mma_commit_w(&s_full[0]);
        }
        if constexpr (kVT) {
          // dS^T(it) ready (the warps have also read dP^T(it)): dQ^T(it) into the dP^T columns first (the
          // drain reads it while dK(it) runs), then dP^T(it+1) once the drain has released the columns
          { long long t0 = TT_CLK(); mbar_wait(&ds_ready[b], (it >> 1) & 1); w_sm += TT_CLK() - t0; }
          tc_fence_after();
          issue_dQ(dsb);
          mma_commit_w(&dq_full[0]);
          const bool dk_first = !(dev_dbg(p.order) & 1);  // dev A/B (TT_BWD_ORDER=1): dP(i+1) before dK(i)
          if (dk_first) {
            issue_dK(dsb, qb, it);
            mma_commit_w(&q_empty[s]);
          }
          if (it + 1 < n_it) {
            { long long t0 = TT_CLK(); mbar_wait(&dq_free[0], it & 1); w_dq += TT_CLK() - t0; }
            tc_fence_after();
            issue_dP(it + 1);
            mma_commit_w(dp_full);
          }
          if (!dk_first) {
            issue_dK(dsb, qb, it);
            mma_commit_w(&q_empty[s]);
          }
          continue;
        }
        // next tile's dP^T (single buffer) as soon as the warps have read dP^T(it)
        if (it + 1 < n_it) {
          { long long t0 = TT_CLK(); mbar_wait(dp_free, it & 1); w_sm += TT_CLK() - t0; }
          tc_fence_after();
          issue_dP(it + 1);
          mma_commit_w(dp_full);
        }
        { long long t0 = TT_CLK(); mbar_wait(&ds_ready[b], (it >> 1) & 1); w_sm += TT_CLK() - t0; }
        tc_fence_after();
        issue_dK(dsb, qb, it);
        if (it > 0) {
          { long long t0 = TT_CLK(); mbar_wait(&dq_free[0], (it - 1) & 1); w_dq += TT_CLK() - t0; }
          tc_fence_after();
        }
        issue_dQ(dsb);
        mma_commit_w(&dq_full[0]);
        mma_commit_w(&q_empty[s]);
        // S^T(it+2) into S^T[b] (in issue order after dV(it) read P^T(it) from it)
        if (!kKT && it + 2 < n_it) {
          { long long t0 = TT_CLK(); mbar_wait(&q_full[(it + 2) % kQStages], ((it + 2) / kQStages) & 1); w_q += TT_CLK() - t0; }
          tc_fence_after();
          issue_SP(it + 2);
          mma_commit_w(&s_full[b]);
        }
      }
      mma_commit_w(acc_done);
      if ((dev_dbg(p.dbg) & 8) && lane == 0) {
        atomicAdd(&g_bwd_dbg[0], (unsigned long long)(TT_CLK() - t_start));
        atomicAdd(&g_bwd_dbg[1], (unsigned long long)w_sm);
        atomicAdd(&g_bwd_dbg[2], (unsigned long long)w_dq);
        atomicAdd(&g_bwd_dbg[3], (unsigned long long)w_q);
        atomicAdd(&g_bwd_dbg[4], (unsigned long long)n_it);
      }
    }
  } else if (warp >= kDrainWarp0) {
    // ===================== dQ drain warpgroup =====================
    const int q4 = warp & 3;
    const int r = q4 * 32 + lane;                      // head-dim lane of dQ^T
    const uint32_t tl = tmem + ((uint32_t)(q4 * 32) << 16);
    long long c_wd = 0, c_dr = 0;
    if constexpr (kKT) {
      // K row (key k0 + r) -> TMEM lane r, columns kColK.. as packed bf16 pairs along d: the A-operand
      // layout of a TS MMA (same packing as P^T)
      const int64_t jr = k0 + r;
      uint32_t kv[64];
      if (jr < p.N) {
        const uint4* src = reinterpret_cast<const uint4*>(p.kmat + (jr * p.hkv + hk) * kD);
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const uint4 x = src[u];
          kv[4 * u] = x.x; kv[4 * u + 1] = x.y; kv[4 * u + 2] = x.z; kv[4 * u + 3] = x.w;
        }
      } else {
#pragma unroll
        for (int u = 0; u < 64; ++u) kv[u] = 0u;
      }
      tmem_st32(tl + kColK, *reinterpret_cast<const uint32_t(*)[32]>(&kv[0]));
      tmem_st32(tl + kColK + 32, *reinterpret_cast<const uint32_t(*)[32]>(&kv[32]));
      if constexpr (kVT) {
        // V row (key k0 + r) -> TMEM lane r, columns kColV.. (A operand of the TS MMA dP^T = V dO^T)
        tmem_wait_st();
        if (jr < p.N) {
          const uint4* src = reinterpret_cast<const uint4*>(p.vmat + (jr * p.hkv + hk) * kD);
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            const uint4 x = src[u];
            kv[4 * u] = x.x; kv[4 * u + 1] = x.y; kv[4 * u + 2] = x.z; kv[4 * u + 3] = x.w;
          }
        }
        tmem_st32(tl + kColV, *reinterpret_cast<const uint32_t(*)[32]>(&kv[0]));
        tmem_st32(tl + kColV + 32, *reinterpret_cast<const uint32_t(*)[32]>(&kv[32]));
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(k_tmem);
    }
    Walk wk;
    for (int it = 0; it < n_it; ++it) {
      int h, q0;
      bwd_item(p, it, wk, nq, qt0, hk, h, q0);
      { long long t0 = TT_CLK(); mbar_wait_role(&dq_full[0], it & 1, dev_dbg(p.wait) & 2); c_wd += TT_CLK() - t0; }
      long long t_dr = TT_CLK();
      tc_fence_after();
      uint32_t v0[32], v1[32];
      tmem_ld32(tl + kColQ, v0);
      tmem_ld32(tl + kColQ + 32, v1);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(&dq_free[0]);
      if (dev_dbg(p.dbg) & 1) continue;
      if ((dev_dbg(p.dbg) & 16) && !TT_DQ_HND) {  // ([N][hq][d] indexing)
        // variant: coalesced fp32 REDs straight from registers (a warp instruction covers 32
        // consecutive head dims of one query row = 128 contiguous bytes); no shared-memory staging
        float* base = p.dq_acc + ((int64_t)q0 * p.hq + h) * kD + r;
        const int64_t rs = (int64_t)p.hq * kD;
        const int nv = (int)imin64(64, p.N - q0);
#pragma unroll
        for (int c = 0; c < 32; ++c)
          if (c < nv) red_add_f32(base + c * rs, __uint_as_float(v0[c]) * p.scale);
#pragma unroll
        for (int c = 0; c < 32; ++c)
          if (32 + c < nv) red_add_f32(base + (32 + c) * rs, __uint_as_float(v1[c]) * p.scale);
        c_dr += TT_CLK() - t_dr;
        continue;
      }
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        // stage hh holds query rows [q0 + 32 hh, +32) x 128 dims ([row][dim], scaled fp32); its previous
        // reduction (one half-tile earlier in issue order) must have finished reading it
        float* stg = reinterpret_cast<float*>(smem + kOffDQ + hh * kDQStage);
        if (r == 0) bulk_wait_read<1>();
        named_bar_sync(1, 128);
        const uint32_t* vv = hh ? v1 : v0;
#pragma unroll
        for (int c = 0; c < 32; ++c) stg[c * kD + r] = __uint_as_float(vv[c]) * p.scale;
        fence_proxy_async_smem();
        named_bar_sync(1, 128);
        if (r == 0) {
          const int hint = dev_dbg(p.l2hint);
          if (dev_dbg(p.dbg) & 32) {
            // dbg 32: staging only
          } else if (hint & 3) {
            tma_reduce_add_3d_hint(&tmdQ, stg, 0, TT_DQ_HND ? q0 + 32 * hh : h, TT_DQ_HND ? h : q0 + 32 * hh, (hint & 1) ? policy_evict_last() : policy_evict_first());
          } else {
            tma_reduce_add_3d(&tmdQ, stg, 0, TT_DQ_HND ? q0 + 32 * hh : h, TT_DQ_HND ? h : q0 + 32 * hh);
          }
          bulk_commit();
        }
      }
      c_dr += TT_CLK() - t_dr;
    }
    if (r == 0) bulk_wait<0>();
    if ((dev_dbg(p.dbg) & 8) && r == 0) {
      atomicAdd(&g_bwd_dbg[7], (unsigned long long)c_dr);
      atomicAdd(&g_bwd_dbg[8], (unsigned long long)c_wd);
    }
  } else {
    // ===================== element-wise warps 2 .. kDrainWarp0-1 =====================
    // kNWG warpgroups share every TMEM lane quadrant (lane quadrant = warp % 4): warpgroup wg owns
    // query columns [kCW wg, kCW wg + kCW) of each 64-row tile.  One thread = one key row.  Measured
    // (role counters, profiles/r1f_bwd_counters_ktmem.txt): with 2 warpgroups (32 columns per thread)
    // these warps were busy ~85% of a tile and latency-bound; 4 warpgroups halve each thread's chain.
    const int wg = (warp - 2) >> 2;
    const int q4 = warp & 3;
    const int r = q4 * 32 + lane;
    const int j = (int)k0 + r;
    const int Nn = (int)p.N;
    const uint32_t tl = tmem + ((uint32_t)(q4 * 32) << 16);
    const int Ej = (j < Nn) ? p.E[j] : -1;
    const float sl2 = p.scale_log2;
    constexpr uint32_t kFull = kCW == 32 ? 0xffffffffu : ((1u << kCW) - 1u);
    long long c_ws = 0, c_el = 0, c_ld = 0, c_math = 0, c_st = 0;
    Walk wk;
    for (int it = 0; it < n_it; ++it) {
      const int s = it % kQStages, b = it & 1;
      int h_unused, q0;
      bwd_item(p, it, wk, nq, qt0, hk, h_unused, q0);
      const int sb = kKT ? 0 : b;
      { long long t0 = TT_CLK(); mbar_wait_role(&s_full[sb], kKT ? (it & 1) : ((it >> 1) & 1), dev_dbg(p.wait) & 2); c_ws += TT_CLK() - t0; }
      tc_fence_after();
      long long t_el = TT_CLK();
      if (dev_dbg(p.dbg) & 4) {
        tc_fence_before();
        mbar_arrive(&p_ready[sb]);
        mbar_wait(dp_full, it & 1);
        tc_fence_after();
        tc_fence_before();
        if constexpr (!kVT) mbar_arrive(dp_free);
        mbar_arrive(&ds_ready[b]);
      } else {
        const float4* st_lse = reinterpret_cast<const float4*>(smem + kOffStats + s * kStatBytes);
        const float4* st_D = reinterpret_cast<const float4*>(smem + kOffStats + s * kStatBytes + 256);
        const float4* st_w = reinterpret_cast<const float4*>(smem + kOffStats + s * kStatBytes + 512);
        const int c0 = q0 + kCW * wg;
        // allowed query columns of this key form one interval: [max(j, c0), min(E_j, N)) - c0
        const int lo = max(j - c0, 0), hi = min(min(Ej, Nn) - c0, kCW);
        const uint32_t cmask = (hi <= lo) ? 0u : ((hi >= kCW ? kFull : ((1u << hi) - 1u)) & ~((1u << lo) - 1u));
        const bool all_in = __all_sync(0xffffffffu, cmask == kFull);
        const float2 SL = make_float2(sl2, sl2);
        // ---- phase P (S^T only): pw = w P, P^T -> TMEM as bf16 ----
        float2 pw[kCW / 2];
        {
          uint32_t sv[kCW], pwk[kCW / 2];
          long long tA = TT_CLK();
          if constexpr (kCW == 32)
            tmem_ld32(tl + kColS + 64 * sb + kCW * wg, *reinterpret_cast<uint32_t(*)[32]>(&sv[0]));
          else
            tmem_ld16(tl + kColS + 64 * sb + kCW * wg, *reinterpret_cast<uint32_t(*)[16]>(&sv[0]));
          tmem_wait_ld();
          c_ld += TT_CLK() - tA;
          tA = TT_CLK();
#pragma unroll
          for (int c4 = 0; c4 < kCW / 4; ++c4) {
            const int cg = (kCW / 4) * wg + c4;  // float4 group within the 64 columns
            const float4 NL = st_lse[cg];  // -LSE * log2e (FOLD: + log2 w)
            const float4 W = FOLD ? make_float4(1.f, 1.f, 1.f, 1.f) : st_w[cg];
            const int c = 4 * c4;
            // P = 2^(s * scale * log2e - LSE2): columns c, c+1 on the MUFU, c+2, c+3 on the FMA pipe
            const float2 a01 = ffma2(make_float2(__uint_as_float(sv[c]), __uint_as_float(sv[c + 1])), SL, make_float2(NL.x, NL.y));
            const float2 a23 = ffma2(make_float2(__uint_as_float(sv[c + 2]), __uint_as_float(sv[c + 3])), SL, make_float2(NL.z, NL.w));
            float2 p01 = make_float2(ex2(a01.x), ex2(a01.y));
#ifndef TT_BWD_POLY
#define TT_BWD_POLY 1
#endif
            // 2 x TT_BWD_POLY of every 8 exponentials run on the FMA pipe
            float2 p23 = (TT_BWD_POLY == 2 || (TT_BWD_POLY == 1 && (c4 & 1))) ? exp2_poly2(a23)
                                                                             : make_float2(ex2(a23.x), ex2(a23.y));
            if (!all_in) {
              p01.x = ((cmask >> c) & 1u) ? p01.x : 0.f;
              p01.y = ((cmask >> (c + 1)) & 1u) ? p01.y : 0.f;
              p23.x = ((cmask >> (c + 2)) & 1u) ? p23.x : 0.f;
              p23.y = ((cmask >> (c + 3)) & 1u) ? p23.y : 0.f;
            }
            if constexpr (FOLD) {
              pw[2 * c4] = p01;
              pw[2 * c4 + 1] = p23;
            } else {
              pw[2 * c4] = fmul2(p01, make_float2(W.x, W.y));
              pw[2 * c4 + 1] = fmul2(p23, make_float2(W.z, W.w));
            }
            pwk[2 * c4] = pack_bf16(pw[2 * c4].x, pw[2 * c4].y);
            pwk[2 * c4 + 1] = pack_bf16(pw[2 * c4 + 1].x, pw[2 * c4 + 1].y);
          }
          // P^T (bf16) over this warpgroup's own S^T columns [kCW wg, kCW wg + kCW / 2) — never over
          // columns another warpgroup may still be reading
          if constexpr (kCW == 32)
            tmem_st16(tl + kColS + 64 * sb + kCW * wg, pwk);
          else
            tmem_st8(tl + kColS + 64 * sb + kCW * wg, pwk);
          tmem_wait_st();
          tc_fence_before();
          mbar_arrive(&p_ready[sb]);
          c_math += TT_CLK() - tA;
        }
        // ---- phase dS (dP^T): dS^T = pw (dP - D) -> smem ----
        {
          uint32_t pv[kCW], dsk[kCW / 2];
          long long tA = TT_CLK();
          { long long t0 = TT_CLK(); mbar_wait_role(dp_full, it & 1, dev_dbg(p.wait) & 2); c_ws += TT_CLK() - t0; }
          tc_fence_after();
          if constexpr (kCW == 32)
            tmem_ld32(tl + kColP + kCW * wg, *reinterpret_cast<uint32_t(*)[32]>(&pv[0]));
          else
            tmem_ld16(tl + kColP + kCW * wg, *reinterpret_cast<uint32_t(*)[16]>(&pv[0]));
          tmem_wait_ld();
          tc_fence_before();
          if constexpr (!kVT) mbar_arrive(dp_free);  // VTMEM: ds_ready (below) releases dP^T's columns
#pragma unroll
          for (int c4 = 0; c4 < kCW / 4; ++c4) {
            const float4 ND = st_D[(kCW / 4) * wg + c4];  // -D
            const int c = 4 * c4;
            const float2 ds01 = fmul2(pw[2 * c4], fadd2(make_float2(__uint_as_float(pv[c]), __uint_as_float(pv[c + 1])), make_float2(ND.x, ND.y)));
            const float2 ds23 = fmul2(pw[2 * c4 + 1], fadd2(make_float2(__uint_as_float(pv[c + 2]), __uint_as_float(pv[c + 3])), make_float2(ND.z, ND.w)));
            dsk[2 * c4] = pack_bf16(ds01.x, ds01.y);
            dsk[2 * c4 + 1] = pack_bf16(ds23.x, ds23.y);
          }
          // dS^T row r into the SWIZZLE_128B smem tile: 16-byte chunk c at (c ^ (r & 7))
          uint8_t* drow = smem + kOffDS + b * kDSTile + r * 128;
#pragma unroll
          for (int c = 0; c < kCW / 8; ++c) {
            const int ch = (kCW / 8) * wg + c;
            *reinterpret_cast<uint4*>(drow + ((ch ^ (r & 7)) << 4)) =
                make_uint4(dsk[4 * c], dsk[4 * c + 1], dsk[4 * c + 2], dsk[4 * c + 3]);
          }
          fence_proxy_async_smem();
          mbar_arrive(&ds_ready[b]);
          c_st += TT_CLK() - tA;
        }
      }
      c_el += TT_CLK() - t_el;
    }
    if ((dev_dbg(p.dbg) & 8) && r == 0 && wg == 0) {
      atomicAdd(&g_bwd_dbg[5], (unsigned long long)c_ws);
      atomicAdd(&g_bwd_dbg[6], (unsigned long long)c_el);
      atomicAdd(&g_bwd_dbg[9], (unsigned long long)c_ld);
      atomicAdd(&g_bwd_dbg[10], (unsigned long long)c_math);
      atomicAdd(&g_bwd_dbg[11], (unsigned long long)c_st);
    }
    // ---- epilogue: the first kNWG/2 warpgroups write dV, the others dK (scaled), each its share of
    //      this key row's 128 head dims ----
    mbar_wait_role(acc_done, 0, dev_dbg(p.wait) & 4);
    tc_fence_after();
    {
      constexpr int kPer = kNWG / 2;              // warpgroups per tensor
      constexpr int kCols = 128 / kPer;           // head dims per warpgroup
      const int tsr = wg / kPer, part = wg % kPer;  // tensor 0 = dV, 1 = dK
      const uint32_t col = (tsr == 0 ? kColDV : kColDK) + kCols * part;
      const float mul = tsr == 0 ? 1.f : p.scale;
      __nv_bfloat16* dst = (tsr == 0 ? p.dv : p.dk) + ((int64_t)j * p.hkv + hk) * kD + kCols * part;
      double sq = 0.0;  // a6: sum of squares of the stored (bf16-rounded) values, fp32 per 8 / fp64 across
#pragma unroll 1
      for (int cc = 0; cc < kCols / 32; ++cc) {
        uint32_t ov[32];
        tmem_ld32(tl + col + 32 * cc, ov);
        tmem_wait_ld();
        if (j < Nn) {
          uint32_t pk[16];
#pragma unroll
          for (int u = 0; u < 16; ++u)
            pk[u] = pack_bf16(__uint_as_float(ov[2 * u]) * mul, __uint_as_float(ov[2 * u + 1]) * mul);
          uint4* d4 = reinterpret_cast<uint4*>(dst + 32 * cc);
#pragma unroll
          for (int u = 0; u < 4; ++u) d4[u] = make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
          if (p.part_kv) {
#pragma unroll
            for (int u8 = 0; u8 < 4; ++u8) {
              float s8 = 0.f;
#pragma unroll
              for (int u = 4 * u8; u < 4 * u8 + 4; ++u) {
                const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pk[u]));
                s8 = fmaf(f.x, f.x, fmaf(f.y, f.y, s8));
              }
              sq += (double)s8;
            }
          }
        }
      }
      if (p.part_kv) {
        // fixed-order reduction over the warpgroup's 128 rows -> one fp64 partial per (CTA, tensor)
        double (*red)[4] = reinterpret_cast<double (*)[4]>(smem + kOffRed);
        for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
        if (lane == 0) red[wg][q4] = sq;
        named_bar_sync(2 + tsr, 128 * kPer);
        if (r == 0 && part == 0) {
          double t = 0.0;
          for (int g2 = tsr * kPer; g2 < (tsr + 1) * kPer; ++g2) t += ((red[g2][0] + red[g2][1]) + red[g2][2]) + red[g2][3];
          p.part_kv[2 * (int64_t)blockIdx.x + tsr] = t;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
  if ((dev_dbg(p.dbg) & 8) && threadIdx.x == 0) {
    atomicAdd(&g_bwd_dbg[12], (unsigned long long)(TT_CLK() - t_kernel0));
    atomicAdd(&g_bwd_dbg[13], 1ull);
  }
}
}  // namespace

// Launch of the flat kernel on the persistent path's prepared workspace / tensor maps (attn_sm100_bwd.cu).
tt_status launch_bwd_flat(const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv, const CUtensorMap& mdo,
                          const CUtensorMap& mdq, const tt_packed& pk, int hq, int hkv, int restore, bool fold,
                          float scale, int chunk, const float* L2p, const float* Dp, const float* wf, int64_t Np,
                          float* dq_acc, void* dk, void* dv, double* part_kv, const void* k, const void* v,
                          cudaStream_t st) {
  BwdParams prm;
  prm.N = pk.n_tokens;
  prm.hq = hq;
  prm.hkv = hkv;
  prm.g = hq / hkv;
  prm.nb = pk.n_blk;
  prm.restore = restore ? 1 : 0;
  prm.chunk = chunk;
  prm.wait = prm.order = prm.l2hint = prm.walk = 0;
  {
    const char* e = dev_getenv("TT_DEBUG_BWD");  // development ablations (dev build only)
    prm.dbg = e ? atoi(e) : 0;
  }
  prm.scale = scale;
  prm.scale_log2 = scale * kLog2e;
  prm.E = pk.E;
  prm.kmaxE = pk.kblk_maxE;
  prm.Np = Np;
  prm.L2p = L2p;
  prm.Dp = Dp;
  prm.wf = wf;
  prm.dq_acc = dq_acc;
  prm.dk = static_cast<__nv_bfloat16*>(dk);
  prm.dv = static_cast<__nv_bfloat16*>(dv);
  prm.part_kv = part_kv;
  prm.kmat = static_cast<const __nv_bfloat16*>(k);
  prm.vmat = static_cast<const __nv_bfloat16*>(v);
  auto kern = fold ? tree_attn_bwd_flat_sm100<true> : tree_attn_bwd_flat_sm100<false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
  if (e != cudaSuccess) { set_error("sm100_attn_bwd (flat): smem attribute: %s", cudaGetErrorString(e)); return TT_ERR_CUDA; }
  const unsigned grid = (unsigned)pk.n_blk * hkv;
  kern<<<grid, kBwdThreads, kSmemBytes, st>>>(mq, mk, mv, mdo, mdq, prm);
  count_launch();
  return check_launch("tree_attn_bwd_flat_sm100");
}

}  // namespace tt
