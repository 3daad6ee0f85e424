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
// Design — key-stationary: a work item is a 128-key block kb of one kv head; it walks
// the contiguous query range [128 kb, maxE_kb) (exact: the queries that see key j are [j, E_j)) in
// 64-row query tiles, for every q head of the GQA group.  K and V are resident in TMEM (copied in from
// shared memory with tcgen05.cp; K also stays in shared memory as dQ^T's A operand); dK and dV
// accumulate in TMEM across all of the item's tiles.
// Persistent CTAs: the grid has one CTA per item and the hardware launches them in order, but a running
// CTA takes over the next not-yet-launched CTA's item through cluster launch control, one item ahead,
// so the next item's K/V loads, TMEM copies and first S^T / dP^T MMAs overlap this item's last tiles and
// its dK/dV epilogue (no CTA exit / launch / TMEM allocation between items).
//   warp 0     producer: the item scheduler (CLC) and TMA: K, V of each item; per tile Q_i, dO_i
//              (64 x 128) into a 3-stage ring, plus LSE (log2), D and w of the 64 rows (bulk copies)
//   warp 1     TMEM allocator + MMA issuer (one elected thread).  Per item: K, V -> TMEM (tcgen05.cp).
//              Per tile:
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
//              Epilogue of each item: warpgroup 0 writes dV, warpgroup 1 writes dK.
//   warps 10-13 dQ drain warpgroup (one thread per head-dim lane of dQ^T): per tile it reads the 64
//              query columns of dQ^T from TMEM, releases the columns to the MMA issuer, and adds them
//              into the fp32 dQ accumulator through two 16 KB smem stages (32 query rows x 128 fp32
//              each, [row][dim]) with TMA bulk tensor reductions (cp.reduce.async.bulk.tensor .add.f32).
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
constexpr int kConsumerThreads = kBwdThreads - 32;         // read every item's info (all but the producer)
constexpr uint32_t kKVTile = 128 * kD * 2;     // 32 KB (two 16 KB chunks of 128 rows x 128 B)
constexpr uint32_t kKVChunk = 128 * 64 * 2;    // 16 KB
constexpr uint32_t kQTile = kBQ * kD * 2;      // 16 KB (two 8 KB chunks of 64 rows x 128 B)
constexpr uint32_t kQChunk = kBQ * 64 * 2;     // 8 KB
// K / V slots 0 and 1: item n's K in slot n & 1 (also dQ^T's A operand), its V in the other (source of
// its TMEM copy only)
constexpr uint32_t kOffQS = 2 * kKVTile;                     // stage s: Q at +s*32K, dO at +s*32K+16K
constexpr uint32_t kDSTile = 128 * kBQ * 2;
constexpr uint32_t kOffDS = kOffQS + kQStages * 2 * kQTile;      // dS^T[2], 16 KB each (1024-aligned)
constexpr uint32_t kOffDQ = kOffDS + 2 * kDSTile;                 // dQ staging: 2 stages x 32 rows x 128 fp32
constexpr uint32_t kDQStage = 32 * kD * 4;
constexpr uint32_t kStatBytes = 768;                              // per stage: -LSE2 | -D | w (256 B each)
constexpr uint32_t kOffStats = kOffDQ + 2 * kDQStage;
constexpr uint32_t kOffBar = kOffStats + kQStages * kStatBytes;
// k_full, v_full, q_full[3], q_empty[3], s_full, p_ready, ds_ready[2], dq_full, dq_free, dp_full,
// acc_done, acc_free, v_free, k_free, item_full[2], item_empty[2], clc
constexpr uint32_t kNumBars = 2 + 2 * kQStages + 1 + 1 + 2 + 1 + 1 + 1 + 1 + 1 + 2 + 4 + 1;
// the next item is claimed (CLC) when its producer reaches this many tiles before the current item's
// end, and published (info + K load) at kPrepareAhead tiles before it
#ifndef TT_BWD_CLAIM_AHEAD
#define TT_BWD_CLAIM_AHEAD 6
#endif
#ifndef TT_BWD_PREPARE_AHEAD
#define TT_BWD_PREPARE_AHEAD 3
#endif
constexpr int kClaimAhead = TT_BWD_CLAIM_AHEAD, kPrepareAhead = TT_BWD_PREPARE_AHEAD;
constexpr uint32_t kOffMisc = (kOffBar + kNumBars * 8 + 15) & ~15u;  // [0] TMEM base
constexpr uint32_t kOffInfo = kOffMisc + 16;                     // item buffers [2]: {item, kb, hk, nq} (item -1: done)
constexpr uint32_t kOffClc = kOffInfo + 2 * 16;                  // cluster-launch-control response
// The dynamic shared-memory window is 1024-byte aligned on sm_100 (checked at run time; the kernel
// traps otherwise), so no alignment slack is reserved.
constexpr uint32_t kOffRed = kOffClc + 16;                        // a6 reduction scratch: double [kNWG][4]
// (no static __shared__ in this kernel: it would shift the 1024-byte aligned dynamic window)
constexpr uint32_t kSmemBytes = kOffRed + 32 * kNWG;
static_assert(kSmemBytes <= 232448, "backward kernel exceeds 227 KB of shared memory");

// TMEM columns: dV 0-127 | dK 128-255 | S^T 256-319 | K 320-383 | dP^T, then dQ^T 384-447 | V 448-511
constexpr uint32_t kColDV = 0, kColDK = 128, kColS = 256, kColK = 320, kColP = 384, kColQ = 384, kColV = 448;

// development instrumentation (TT_DEBUG_BWD & 8): per-role cycle counters summed over CTAs
__device__ unsigned long long g_bwd_dbg[16];

struct BwdParams {
  int64_t N;
  int hq, hkv, g, nb;
  int restore;
  int chunk;  // CTA order: key blocks in chunks of `chunk`; within a chunk the kv heads outermost (1 = heads
              // fastest, >= nb = head-major: the Q / dO / dQ rows of one head group stay L2-resident)
  int steal;  // persistent CTAs: take over not-yet-launched CTAs' items (dev A/B TT_BWD_NOSTEAL: 0)
  int wait;   // dev A/B (TT_WAIT_HINT): suspend-hint waits, bit 0 producer, 1 consumers, 2 epilogue
  int dbg;    // development ablations (TT_DEBUG_BWD): 1 skip dQ reduce, 4 skip elementwise math, 8 counters,
              // 32 stage dQ but skip the L2 reduce
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
  double* part_kv;  // nullable: [grid][2] fp64 partial sums of squares of an item's dV (0) / dK (1) rows
};

// work item x (a blockIdx.x of the grid) -> (key block, kv head) and its number of 64-row query tiles
__device__ __forceinline__ int4 bwd_item_of(const BwdParams& p, int x) {
  const int per = p.chunk * p.hkv;
  const int ch = x / per, w = x - ch * per;
  const int len = min(p.chunk, p.nb - ch * p.chunk);
  const int hk = w / len;
  const int kb = ch * p.chunk + (w - hk * len);
  const int nq = (int)((p.kmaxE[kb] + kBQ - 1) / kBQ) - 2 * kb;  // query tiles [2 kb, ceil(maxE / 64))
  return make_int4(x, kb, hk, nq);
}

// tile `it` of an item -> (q head, first query row): GQA heads outer, query tiles ascending, advanced
// with a (tile, head) counter pair (no integer division per tile)
struct Walk {
  int qi = 0, hi = 0;
  __device__ __forceinline__ void next(const BwdParams& p, int nq, int kb, int hk, int& h, int& q0) {
    h = hk * p.g + hi;
    q0 = (2 * kb + qi) * kBQ;
    if (++qi == nq) { qi = 0; ++hi; }
  }
};

// FOLD: the tree-scale is folded into the preprocessed LSE (L2p = -LSE log2e + log2 w, valid for w >= 0:
// integer trajectory counts, non-negative real weights, or restore off), so P w = exp2(s scale log2e + L2p)
// costs no multiply and no per-tile load of w; real-valued weights with some w < 0 take the multiply.
template <bool FOLD>
__global__ void __maxnreg__(kNWG == 4 ? 80 : 128)  // 22 warps: 6 per SMSP x 80 regs x 32 fit its 16K registers
    tree_attn_bwd_sm100(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                        const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmdO,
                        const __grid_constant__ CUtensorMap tmdQ, const BwdParams p) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned base; pointer arithmetic on smem_raw keeps the shared address space visible to
  // the compiler (LDS/STS instead of generic LD/ST)
  uint8_t* smem = smem_raw;
  if (smem_u32(smem_raw) & 1023u) __trap();
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar);
  uint64_t* k_full = bars;                // K of the item in shared memory
  uint64_t* v_full = bars + 1;            // V of the item in shared memory
  uint64_t* q_full = bars + 2;
  uint64_t* q_empty = q_full + kQStages;
  uint64_t* s_full = q_empty + kQStages;  // S^T(i) in TMEM
  uint64_t* p_ready = s_full + 1;         // P^T(i) packed back into S^T (128 kNWG arrivals)
  uint64_t* ds_ready = p_ready + 1;       // [2] dS^T(i) in smem (128 kNWG arrivals)
  uint64_t* dq_full = ds_ready + 2;       // dQ^T(i) in TMEM
  uint64_t* dq_free = dq_full + 1;        // dQ^T(i) read by the drain (128 arrivals)
  uint64_t* dp_full = dq_free + 1;        // dP^T(i) in TMEM
  uint64_t* acc_done = dp_full + 1;       // the item's dK / dV final
  uint64_t* acc_free = acc_done + 1;      // the item's dK / dV read out of TMEM (128 drain arrivals)
  uint64_t* v_free = acc_free + 1;        // the item's V TMEM copy done (V's smem slot free)
  uint64_t* k_free = v_free + 1;          // the item's last dQ^T done (K's smem slot free)
  uint64_t* item_full = k_free + 1;       // [2] item info written
  uint64_t* item_empty = item_full + 2;   // [2] item info read (every consumer thread)
  uint64_t* clc_bar = item_empty + 2;
  uint32_t* misc = reinterpret_cast<uint32_t*>(smem + kOffMisc);
  int4* info = reinterpret_cast<int4*>(smem + kOffInfo);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long t_kernel0 = TT_CLK();

  if (warp == 1) {
    if (lane == 0) {
      mbar_init(k_full, 1);
      mbar_init(v_full, 1);
      mbar_init(acc_free, 128);
      for (int s = 0; s < kQStages; ++s) { mbar_init(&q_full[s], 1); mbar_init(&q_empty[s], 1); }
      mbar_init(s_full, 1);
      mbar_init(p_ready, 128 * kNWG);
      for (int b = 0; b < 2; ++b) mbar_init(&ds_ready[b], 128 * kNWG);
      mbar_init(dq_full, 1);
      mbar_init(dq_free, 128);
      mbar_init(dp_full, 1);
      mbar_init(acc_done, 1);
      mbar_init(v_free, 1);
      mbar_init(k_free, 1);
      for (int b = 0; b < 2; ++b) { mbar_init(&item_full[b], 1); mbar_init(&item_empty[b], kConsumerThreads); }
      mbar_init(clc_bar, 1);
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
    // ===================== producer warp: item scheduler (CLC) + TMA =====================
    // An item's K goes to shared-memory slot (n & 1), its V to the other slot: K(n+1) can land in V(n)'s
    // slot as soon as V(n) was copied into TMEM (early in item n), V(n+1) in K(n)'s slot once item n's
    // last dQ^T (K's last reader) completed.
    bool steal = p.steal != 0;
    uint32_t clc_ph = 0;
    if (lane == 0) {
      tma_prefetch(&tmQ);
      tma_prefetch(&tmK);
      tma_prefetch(&tmV);
      tma_prefetch(&tmdO);
    }
    auto load_k = [&](int slot, int kb, int hk) {
      mbar_expect_tx(k_full, kKVTile);
      for (int c = 0; c < 2; ++c) tma_load_3d(smem + slot * kKVTile + c * kKVChunk, &tmK, k_full, c * 64, hk, kb * 128);
    };
    auto load_v = [&](int slot, int kb, int hk) {
      mbar_expect_tx(v_full, kKVTile);
      for (int c = 0; c < 2; ++c) tma_load_3d(smem + slot * kKVTile + c * kKVChunk, &tmV, v_full, c * 64, hk, kb * 128);
    };
    int4 cur = bwd_item_of(p, (int)blockIdx.x);
    if (lane == 0) {
      load_k(0, cur.y, cur.z);
      load_v(1, cur.y, cur.z);
      info[0] = cur;
      mbar_arrive(&item_full[0]);
    }
    uint32_t G = 0;  // query tiles issued so far (all items): stage G % kQStages
    for (int n = 0;; ++n) {
      const int kb = cur.y, hk = cur.z, nq = cur.w, n_it = nq * p.g;
      // V(n) (n >= 1) goes into K(n-1)'s slot once item n-1's last dQ^T completed; that dQ^T is issued
      // after item n's first S^T, so the wait comes after this item's first Q / dO load
      int4 nxt = make_int4(-1, 0, 0, 0);
      bool claimed = false, prepared = false;
      // The next item is claimed late (a few tiles before this one ends: claiming at the start of an
      // item would pair heavy items on one CTA and unbalance the tail) and published with its K load
      // once this item's last Q / dO tiles are in flight.
      auto claim = [&]() {
        claimed = true;
        if (steal && lane == 0) {
          mbar_expect_tx(clc_bar, 16);
          clc_try_cancel(smem + kOffClc, clc_bar);
        }
      };
      auto prepare_next = [&]() {
        prepared = true;
        if (!claimed) claim();
        if (steal) {
          mbar_wait(clc_bar, clc_ph);
          clc_ph ^= 1;
          const int xn = clc_query_x(smem + kOffClc);
          fence_proxy_async_smem();
          __syncwarp();
          if (xn < 0) steal = false;  // no further request after a failed one
          else nxt = bwd_item_of(p, xn);
        }
        if (n >= 1) mbar_wait(&item_empty[(n + 1) & 1], ((n - 1) >> 1) & 1);  // item n-1's info read
        if (lane == 0) {
          info[(n + 1) & 1] = nxt;
          mbar_arrive(&item_full[(n + 1) & 1]);
        }
        if (nxt.x >= 0) {
          mbar_wait(v_free, n & 1);  // V(n) copied into TMEM: its slot takes K(n+1)
          if (lane == 0) load_k((n + 1) & 1, nxt.y, nxt.z);
        }
      };
      Walk wk;
      for (int it = 0; it < n_it; ++it, ++G) {
        const int s = (int)(G % kQStages);
        if (G >= (uint32_t)kQStages) mbar_wait_role(&q_empty[s], ((G / kQStages) - 1) & 1, dev_dbg(p.wait) & 1);
        int h, q0;
        wk.next(p, nq, kb, hk, h, q0);
        if (lane == 0) {
          uint8_t* qd = smem + kOffQS + s * 2 * kQTile;
          uint8_t* st = smem + kOffStats + s * kStatBytes;
          mbar_expect_tx(&q_full[s], 2 * kQTile + 3 * 256);
          for (int c = 0; c < 2; ++c) {
            tma_load_3d(qd + c * kQChunk, &tmQ, &q_full[s], c * 64, h, q0);
            tma_load_3d(qd + kQTile + c * kQChunk, &tmdO, &q_full[s], c * 64, h, q0);
          }
          bulk_load_1d(st, p.L2p + (int64_t)h * p.Np + q0, 256, &q_full[s]);
          bulk_load_1d(st + 256, p.Dp + (int64_t)h * p.Np + q0, 256, &q_full[s]);
          bulk_load_1d(st + 512, p.wf + q0, 256, &q_full[s]);
        }
        if (it == 0 && n >= 1) {
          mbar_wait(k_free, (n - 1) & 1);
          if (lane == 0) load_v((n - 1) & 1, kb, hk);
        }
        if (!claimed && it >= n_it - kClaimAhead) claim();
        if (!prepared && it >= n_it - kPrepareAhead) prepare_next();
      }
      if (!prepared) prepare_next();
      if (nxt.x < 0) break;
      cur = nxt;
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (whole warp, one elected lane issues) =====================
    // One stream of query tiles across items: the last tile of item n issues item n+1's K copy and
    // first S^T in place of "S(i+1)", and its V copy and first dP^T in place of "dP(i+1)", so the tensor
    // pipe runs on while item n's dK / dV are read out by the drain warpgroup; item n+1's first dV
    // (which overwrites them) waits for acc_free.
    constexpr uint32_t idSP = idesc_bf16(128, kBQ, 0, 0);   // K/V (TMEM) x Q/dO^T (K-major)
    constexpr uint32_t idVK = idesc_bf16(128, 128, 0, 1);   // P^T/dS^T (K-major) x dO/Q (MN-major)
    constexpr uint32_t idQ = idesc_bf16(128, kBQ, 1, 1);    // K^T (MN-major) x dS^T (MN-major)
    const uint32_t sm0 = warp_uniform(smem_u32(smem));
    const uint32_t tm = warp_uniform(tmem);
    const uint32_t qs0 = sm0 + kOffQS, ds0 = sm0 + kOffDS;
    auto issue_S = [&](uint32_t Gi) {
      const uint32_t qb = qs0 + (Gi % kQStages) * 2 * kQTile;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t offq = (kk >> 2) * kQChunk + (kk & 3) * 32;
        mma_ts_w(tm + kColS, tm + kColK + 8 * kk, sdesc(qb + offq, 16, 1024), idSP, kk > 0);
      }
    };
    auto issue_dP = [&](uint32_t Gi) {
      const uint32_t ob = qs0 + (Gi % kQStages) * 2 * kQTile + kQTile;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t offq = (kk >> 2) * kQChunk + (kk & 3) * 32;
        mma_ts_w(tm + kColP, tm + kColV + 8 * kk, sdesc(ob + offq, 16, 1024), idSP, kk > 0);
      }
    };
    // K or V (128 keys x 128 dims, SWIZZLE_128B K-major in shared memory) -> TMEM (TS-MMA A layout)
    auto copy_in = [&](uint32_t col, uint32_t src) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        tmem_cp_w(tm + col + 8 * kk, sdesc(src + (kk >> 2) * kKVChunk + (kk & 3) * 32, 16, 1024));
    };
    // dQ^T = K^T dS^T   (A: K MN-major, LBO = 16 KB d-chunk; B: dS^T MN-major, one 64-wide group)
    auto issue_dQ = [&](uint32_t ksb, uint32_t dsb) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        mma_ss_w(tm + kColQ, sdesc(ksb + kk * 2048, kKVChunk, 1024), sdesc(dsb + kk * 2048, kDSTile, 1024),
                 idQ, kk > 0);
    };
    // dK += dS^T Q   (A: dS^T K-major 128 x 64 in smem; B: Q MN-major)
    auto issue_dK = [&](uint32_t dsb, uint32_t qb, int it) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        mma_ss_w(tm + kColDK, sdesc(dsb + kk * 32, 16, 1024), sdesc(qb + kk * 2048, kQChunk, 1024), idVK,
                 (it > 0 || kk > 0) ? 1u : 0u);
    };
    long long w_sm = 0, w_dq = 0, w_q = 0, w_item = 0, t_start = TT_CLK();
    uint32_t G = 0;  // query tiles consumed so far (all items)
    int n_items = 0;
    mbar_wait(&item_full[0], 0);
    int4 cur = info[0];
    mbar_arrive(&item_empty[0]);
    // item 0: K, V -> TMEM, S(0), dP(0)
    mbar_wait(k_full, 0);
    tc_fence_after();
    copy_in(kColK, sm0 + 0 * kKVTile);
    mbar_wait(&q_full[0], 0);
    tc_fence_after();
    issue_S(0);
    mma_commit_w(s_full);
    mbar_wait(v_full, 0);
    tc_fence_after();
    copy_in(kColV, sm0 + 1 * kKVTile);
    mma_commit_w(v_free);
    issue_dP(0);
    mma_commit_w(dp_full);
    for (int n = 0;; ++n) {
      const int n_it = cur.w * p.g;
      const uint32_t ksb = sm0 + (n & 1) * kKVTile;  // this item's K slot
      int4 nxt = make_int4(-1, 0, 0, 0);
      ++n_items;
      for (int it = 0; it < n_it; ++it) {
        const uint32_t Gi = G + (uint32_t)it;
        const uint32_t s = Gi % kQStages;
        const uint32_t qb = qs0 + s * 2 * kQTile;
        const uint32_t ob = qb + kQTile;
        const uint32_t dsb = ds0 + (Gi & 1) * kDSTile;
        const bool last = it + 1 == n_it;
        { long long t0 = TT_CLK(); mbar_wait(p_ready, Gi & 1); w_sm += TT_CLK() - t0; }
        if (it == 0 && n > 0) {  // the drain warpgroup has read item n-1's dK / dV out of TMEM
          const long long t0 = TT_CLK();
          mbar_wait(acc_free, (n - 1) & 1);
          w_item += TT_CLK() - t0;
        }
        tc_fence_after();
        // dV += P^T dO   (A: P^T bf16 in TMEM over S^T; B: dO MN-major, LBO = 8 KB d-chunk)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)  // P^T of query columns 16 kk.. : warpgroup 16 kk / kCW packed it at its own S^T columns
          mma_ts_w(tm + kColDV, tm + kColS + kCW * ((16 * kk) / kCW) + 8 * (((16 * kk) % kCW) / 16),
                   sdesc(ob + kk * 2048, kQChunk, 1024), idVK, (it > 0 || kk > 0) ? 1u : 0u);
        // the single S^T buffer takes the next tile's S^T right after dV(i) has read P^T(i) from it
        if (last) {
          mbar_wait(&item_full[(n + 1) & 1], ((n + 1) >> 1) & 1);
          nxt = info[(n + 1) & 1];
          mbar_arrive(&item_empty[(n + 1) & 1]);
          if (nxt.x >= 0) {  // item n+1's K -> TMEM (item n's S^T MMAs, its readers, are complete)
            const long long t0 = TT_CLK();
            mbar_wait(k_full, (n + 1) & 1);
            w_item += TT_CLK() - t0;
            tc_fence_after();
            copy_in(kColK, sm0 + ((n + 1) & 1) * kKVTile);
          }
        }
        if (!last || nxt.x >= 0) {
          { long long t0 = TT_CLK(); mbar_wait(&q_full[(Gi + 1) % kQStages], ((Gi + 1) / kQStages) & 1); w_q += TT_CLK() - t0; }
          tc_fence_after();
          issue_S(Gi + 1);
          mma_commit_w(s_full);
        }
        // dS^T(i) ready (the warps have also read dP^T(i)): dQ^T(i) into the dP^T columns first (the
        // drain reads it while dK(i) runs), then the next dP^T once the drain has released the columns
        { long long t0 = TT_CLK(); mbar_wait(&ds_ready[Gi & 1], (Gi >> 1) & 1); w_sm += TT_CLK() - t0; }
        tc_fence_after();
        issue_dQ(ksb, dsb);
        mma_commit_w(dq_full);
        if (last) mma_commit_w(k_free);  // the item's last reader of K in shared memory
        issue_dK(dsb, qb, it);
        mma_commit_w(&q_empty[s]);
        if (last) mma_commit_w(acc_done);  // item n's dK / dV final
        if (last && nxt.x >= 0) {  // item n+1's V -> TMEM (item n's dP^T MMAs, its readers, are complete)
          const long long t0 = TT_CLK();
          mbar_wait(v_full, (n + 1) & 1);
          w_item += TT_CLK() - t0;
          tc_fence_after();
          copy_in(kColV, sm0 + (n & 1) * kKVTile);
          mma_commit_w(v_free);
        }
        if (!last || nxt.x >= 0) {
          { long long t0 = TT_CLK(); mbar_wait(dq_free, Gi & 1); w_dq += TT_CLK() - t0; }
          tc_fence_after();
          issue_dP(Gi + 1);
          mma_commit_w(dp_full);
        }
      }
      G += (uint32_t)n_it;
      if (nxt.x < 0) break;
      cur = nxt;
    }
    if ((dev_dbg(p.dbg) & 8) && lane == 0) {
      atomicAdd(&g_bwd_dbg[0], (unsigned long long)(TT_CLK() - t_start));
      atomicAdd(&g_bwd_dbg[1], (unsigned long long)w_sm);
      atomicAdd(&g_bwd_dbg[2], (unsigned long long)w_dq);
      atomicAdd(&g_bwd_dbg[3], (unsigned long long)w_q);
      atomicAdd(&g_bwd_dbg[4], (unsigned long long)G);
      atomicAdd(&g_bwd_dbg[14], (unsigned long long)w_item);
      atomicAdd(&g_bwd_dbg[15], (unsigned long long)n_items);
    }
  } else if (warp >= kDrainWarp0) {
    // ===================== dQ drain warpgroup (+ each item's dK / dV epilogue) =====================
    const int q4 = warp & 3;
    const int r = q4 * 32 + lane;                      // head-dim lane of dQ^T; key row of dK / dV
    const uint32_t tl = tmem + ((uint32_t)(q4 * 32) << 16);
    const int Nn = (int)p.N;
    long long c_wd = 0, c_dr = 0;
    uint32_t G = 0;
    for (int n = 0;; ++n) {
      mbar_wait(&item_full[n & 1], (n >> 1) & 1);
      const int4 cur = info[n & 1];
      mbar_arrive(&item_empty[n & 1]);
      if (cur.x < 0) break;
      const int nq = cur.w, n_it = nq * p.g;
      Walk wk;
      for (int it = 0; it < n_it; ++it, ++G) {
        int h, q0;
        wk.next(p, nq, cur.y, cur.z, h, q0);
        { long long t0 = TT_CLK(); mbar_wait_role(dq_full, G & 1, dev_dbg(p.wait) & 2); c_wd += TT_CLK() - t0; }
        long long t_dr = TT_CLK();
        tc_fence_after();
        uint32_t v0[32], v1[32];
        tmem_ld32(tl + kColQ, v0);
        tmem_ld32(tl + kColQ + 32, v1);
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive(dq_free);
        if (dev_dbg(p.dbg) & 1) continue;
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
            if (!(dev_dbg(p.dbg) & 32)) tma_reduce_add_3d(&tmdQ, stg, 0, TT_DQ_HND ? q0 + 32 * hh : h, TT_DQ_HND ? h : q0 + 32 * hh);  // dbg 32: staging only
            bulk_commit();
          }
        }
        c_dr += TT_CLK() - t_dr;
      }
      // ---- item epilogue: key row r's dV and dK (scaled) -> bf16 (a6: fp64 sums of squares of the
      //      stored values, fp32 per 8).  acc_free is arrived on once every TMEM read is done, before
      //      the stores drain, so item n+1's first dV / dK MMAs wait only for the reads. ----
      mbar_wait_role(acc_done, n & 1, dev_dbg(p.wait) & 4);
      tc_fence_after();
      const int j = cur.y * 128 + r;
      double sq[2] = {0.0, 0.0};
#pragma unroll
      for (int tsr = 0; tsr < 2; ++tsr) {  // 0 = dV (columns 0-127), 1 = dK (128-255)
        const float mul = tsr == 0 ? 1.f : p.scale;
        __nv_bfloat16* dst = (tsr == 0 ? p.dv : p.dk) + ((int64_t)j * p.hkv + cur.z) * kD;
#pragma unroll 1
        for (int cc = 0; cc < 4; ++cc) {
          uint32_t ov[32];
          tmem_ld32(tl + kColDV + 128 * tsr + 32 * cc, ov);
          tmem_wait_ld();
          if (tsr == 1 && cc == 3) {
            tc_fence_before();
            mbar_arrive(acc_free);
          }
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
                sq[tsr] += (double)s8;
              }
            }
          }
        }
      }
      if (p.part_kv) {
        // fixed-order reduction over the item's 128 key rows -> one fp64 partial per (item, tensor)
        double (*red)[4] = reinterpret_cast<double (*)[4]>(smem + kOffRed);
        for (int t2 = 0; t2 < 2; ++t2)
          for (int o = 16; o > 0; o >>= 1) sq[t2] += __shfl_xor_sync(0xffffffffu, sq[t2], o);
        if (lane == 0) { red[0][q4] = sq[0]; red[1][q4] = sq[1]; }
        named_bar_sync(2, 128);
        if (r == 0)
          for (int t2 = 0; t2 < 2; ++t2)
            p.part_kv[2 * (int64_t)cur.x + t2] = ((red[t2][0] + red[t2][1]) + red[t2][2]) + red[t2][3];
      }
    }
    if (r == 0) bulk_wait<0>();
    if ((dev_dbg(p.dbg) & 8) && r == 0) {
      atomicAdd(&g_bwd_dbg[7], (unsigned long long)c_dr);
      atomicAdd(&g_bwd_dbg[8], (unsigned long long)c_wd);
    }
  } else {
    // ===================== element-wise warps 2 .. kDrainWarp0-1 =====================
    // kNWG warpgroups share every TMEM lane quadrant (lane quadrant = warp % 4): warpgroup wg owns
    // query columns [kCW wg, kCW wg + kCW) of each 64-row tile.  One thread = one key row.
    const int wg = (warp - 2) >> 2;
    const int q4 = warp & 3;
    const int r = q4 * 32 + lane;
    const int Nn = (int)p.N;
    const uint32_t tl = tmem + ((uint32_t)(q4 * 32) << 16);
    const float sl2 = p.scale_log2;
    constexpr uint32_t kFull = kCW == 32 ? 0xffffffffu : ((1u << kCW) - 1u);
    long long c_ws = 0, c_el = 0, c_ld = 0, c_math = 0, c_st = 0;
    uint32_t G = 0;
    for (int n = 0;; ++n) {
      mbar_wait(&item_full[n & 1], (n >> 1) & 1);
      const int4 cur = info[n & 1];
      mbar_arrive(&item_empty[n & 1]);
      if (cur.x < 0) break;
      const int kb = cur.y, hk = cur.z, nq = cur.w, n_it = nq * p.g;
      const int j = kb * 128 + r;
      const int Ej = (j < Nn) ? p.E[j] : -1;
      Walk wk;
      for (int it = 0; it < n_it; ++it, ++G) {
        const int s = (int)(G % kQStages), b = (int)(G & 1);
        int h_unused, q0;
        wk.next(p, nq, kb, hk, h_unused, q0);
        { long long t0 = TT_CLK(); mbar_wait_role(s_full, G & 1, dev_dbg(p.wait) & 2); c_ws += TT_CLK() - t0; }
        tc_fence_after();
        long long t_el = TT_CLK();
        if (dev_dbg(p.dbg) & 4) {
          tc_fence_before();
          mbar_arrive(p_ready);
          mbar_wait(dp_full, G & 1);
          tc_fence_after();
          tc_fence_before();
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
              tmem_ld32(tl + kColS + kCW * wg, *reinterpret_cast<uint32_t(*)[32]>(&sv[0]));
            else
              tmem_ld16(tl + kColS + kCW * wg, *reinterpret_cast<uint32_t(*)[16]>(&sv[0]));
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
              tmem_st16(tl + kColS + kCW * wg, pwk);
            else
              tmem_st8(tl + kColS + kCW * wg, pwk);
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(p_ready);
            c_math += TT_CLK() - tA;
          }
          // ---- phase dS (dP^T): dS^T = pw (dP - D) -> smem ----
          {
            uint32_t pv[kCW], dsk[kCW / 2];
            long long tA = TT_CLK();
            { long long t0 = TT_CLK(); mbar_wait_role(dp_full, G & 1, dev_dbg(p.wait) & 2); c_ws += TT_CLK() - t0; }
            tc_fence_after();
            if constexpr (kCW == 32)
              tmem_ld32(tl + kColP + kCW * wg, *reinterpret_cast<uint32_t(*)[32]>(&pv[0]));
            else
              tmem_ld16(tl + kColP + kCW * wg, *reinterpret_cast<uint32_t(*)[16]>(&pv[0]));
            tmem_wait_ld();
            tc_fence_before();  // ds_ready (below) also releases dP^T's columns to dQ^T
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
    }
    if ((dev_dbg(p.dbg) & 8) && r == 0 && wg == 0) {
      atomicAdd(&g_bwd_dbg[5], (unsigned long long)c_ws);
      atomicAdd(&g_bwd_dbg[6], (unsigned long long)c_el);
      atomicAdd(&g_bwd_dbg[9], (unsigned long long)c_ld);
      atomicAdd(&g_bwd_dbg[10], (unsigned long long)c_math);
      atomicAdd(&g_bwd_dbg[11], (unsigned long long)c_st);
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

// dQ fp32 accumulator -> bf16 output; optionally the per-block fp64 sum of squares of the rounded
// values (fixed grid and grid-stride assignment: bitwise reproducible)
__global__ void __launch_bounds__(256) dq_convert_kernel(const float4* __restrict__ acc, uint2* __restrict__ out,
                                                         int64_t n4, double* __restrict__ part_q, int64_t N, int hq) {
  double sq = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    // output element i = (token, head, 4 dims); TT_DQ_HND reads it from the [hq][N][d] accumulator
    int64_t ia = i;
    if (TT_DQ_HND) {
      const int64_t d4 = i & 31, th = i >> 5, t = th / hq, h = th - t * hq;
      ia = ((int64_t)h * N + t) * 32 + d4;
    }
    const float4 a = acc[ia];
    const uint2 o = make_uint2(pack_bf16(a.x, a.y), pack_bf16(a.z, a.w));
    out[i] = o;
    if (part_q) {
      const float2 lo = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&o.x));
      const float2 hi = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&o.y));
      sq += (double)fmaf(lo.x, lo.x, fmaf(lo.y, lo.y, fmaf(hi.x, hi.x, hi.y * hi.y)));
    }
  }
  if (!part_q) return;
  __shared__ double red[8];
  for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sq;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w];
    part_q[blockIdx.x] = t;
  }
}

// a6: ||dQ||^2, ||dK||^2, ||dV||^2 from the per-block / per-CTA partials, fixed order, one CTA
__global__ void __launch_bounds__(256) sqnorm_final_kernel(const double* __restrict__ part_q, int nq,
                                                           const double* __restrict__ part_kv, int nkv,
                                                           double* __restrict__ out) {
  __shared__ double red[3][256];
  double a = 0.0, b = 0.0, c = 0.0;
  for (int i = threadIdx.x; i < nq; i += 256) a += part_q[i];
  for (int i = threadIdx.x; i < nkv; i += 256) { c += part_kv[2 * i]; b += part_kv[2 * i + 1]; }
  red[0][threadIdx.x] = a;
  red[1][threadIdx.x] = b;
  red[2][threadIdx.x] = c;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w)
      for (int k = 0; k < 3; ++k) red[k][threadIdx.x] += red[k][threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x < 3) out[threadIdx.x] = red[threadIdx.x][0];
}

}  // namespace

extern "C" int tt_debug_bwd_counters(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, g_bwd_dbg, sizeof(g_bwd_dbg));
  if (reset) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(g_bwd_dbg, z, sizeof(z));
  }
  return 0;
}

static inline size_t al256b(size_t x) { return (x + 255) & ~size_t(255); }

constexpr int kDqConvBlocks = 148 * 16;
size_t sm100_bwd_ws_bytes(int64_t N, int hq, int hkv, int d) {
  const int64_t Np = (N + 127) / 128 * 128;
  const int64_t nb = Np / 128;
  return 2 * al256b((size_t)hq * Np * 4) + al256b((size_t)Np * 4) + al256b((size_t)N * hq * d * 4) +
         al256b((size_t)(kDqConvBlocks + 2 * nb * hkv) * sizeof(double));
}

// the non-persistent kernel for long work items (attn_sm100_bwd_flat.cu)
tt_status launch_bwd_flat(const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv, const CUtensorMap& mdo,
                          const CUtensorMap& mdq, const tt_packed& pk, int hq, int hkv, int restore, bool fold,
                          float scale, int chunk, const float* L2p, const float* Dp, const float* wf, int64_t Np,
                          float* dq_acc, void* dk, void* dv, double* part_kv, const void* k, const void* v,
                          cudaStream_t st);

tt_status sm100_attn_bwd(const tt_packed& pk, const void* q, const void* k, const void* v, const void* o,
                         const float* lse, const void* dout, int restore, int hq, int hkv, int d, float scale,
                         void* ws, void* dq, void* dk, void* dv, double* sqnorm, cudaStream_t st) {
  if (d != kD) { set_error("sm100_attn_bwd: d must be 128"); return TT_ERR_UNSUPPORTED; }
  const int64_t N = pk.n_tokens;
  const int64_t Np = (N + 127) / 128 * 128;
  char* w8 = static_cast<char*>(ws);
  float* Dp = reinterpret_cast<float*>(w8);
  float* L2p = reinterpret_cast<float*>(w8 + al256b((size_t)hq * Np * 4));
  float* wf = reinterpret_cast<float*>(w8 + 2 * al256b((size_t)hq * Np * 4));
  float* dq_acc = reinterpret_cast<float*>(w8 + 2 * al256b((size_t)hq * Np * 4) + al256b((size_t)Np * 4));
  double* part_q = reinterpret_cast<double*>(w8 + 2 * al256b((size_t)hq * Np * 4) + al256b((size_t)Np * 4) +
                                             al256b((size_t)N * hq * d * 4));
  double* part_kv = part_q + kDqConvBlocks;
  bool fold = !restore || pk.wr == nullptr || !pk.wr_negative;  // integer trajectory counts are >= 0
  if (dev_getenv("TT_BWD_NOFOLD")) fold = false;  // development A/B: the multiply form
  tt_status s = launch_bwd_pre_tc(o, dout, lse, pk.w, pk.wr, restore, fold ? 1 : 0, N, Np, hq, Dp, L2p, wf, dq_acc, st);
  if (s) return s;
  CUtensorMap mq, mk, mv, mdo, mdq;
  const auto BF = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  const auto SW = CU_TENSOR_MAP_SWIZZLE_128B;
  if ((s = make_tmap_thd(&mq, q, N, hq, d, kBQ, BF, 2, SW, 64))) return s;
  if ((s = make_tmap_thd(&mdo, dout, N, hq, d, kBQ, BF, 2, SW, 64))) return s;
  if ((s = make_tmap_thd(&mk, k, N, hkv, d, 128, BF, 2, SW, 64))) return s;
  if ((s = make_tmap_thd(&mv, v, N, hkv, d, 128, BF, 2, SW, 64))) return s;
  if (TT_DQ_HND) {
    const int64_t dims[3] = {d, N, hq}, strides[2] = {d, N * d};
    const int box[3] = {kD, 32, 1};
    if ((s = make_tmap_3d(&mdq, dq_acc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, dims, strides, box))) return s;
  } else if ((s = make_tmap_thd(&mdq, dq_acc, N, hq, d, 32, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
                                CU_TENSOR_MAP_SWIZZLE_NONE, kD))) {
    return s;
  }
  BwdParams prm;
  prm.N = N;
  prm.hq = hq;
  prm.hkv = hkv;
  prm.g = hq / hkv;
  prm.nb = pk.n_blk;
  prm.restore = restore ? 1 : 0;
  {
    const char* e = dev_getenv("TT_DEBUG_BWD");
    prm.dbg = e ? atoi(e) : 0;
    const char* o = dev_getenv("TT_CTA_ORDER");  // development A/B: bit 1 = bwd head-major
    const char* wh = dev_getenv("TT_WAIT_HINT");
    prm.wait = wh ? atoi(wh) : 0;
    prm.steal = dev_getenv("TT_BWD_NOSTEAL") ? 0 : 1;  // development A/B: one item per CTA
    prm.chunk = bwd_cta_chunk(pk, hkv);
    if (o && ((atoi(o) >> 1) & 1)) prm.chunk = pk.n_blk;  // development A/B: head-major
    if (const char* c = dev_getenv("TT_BWD_CHUNK")) prm.chunk = atoi(c) > 0 ? atoi(c) : 1;
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
  prm.part_kv = sqnorm ? part_kv : nullptr;
  // Long work items (mean query tiles per item >= kBwdFlatMinTilesPerItem, from the pack's host schedule
  // statistics) go to the non-persistent kernel (attn_sm100_bwd_flat.cu): item boundaries are rare there
  // and it measured 1-2% faster per tile; short items (small trees) take the persistent kernel.
  bool flat = bwd_use_flat(pk, hq, hkv);
  if (const char* f = dev_getenv("TT_BWD_FLAT")) flat = atoi(f) != 0;  // development A/B: force either kernel
  if (flat) {
    s = launch_bwd_flat(mq, mk, mv, mdo, mdq, pk, hq, hkv, restore, fold, scale, prm.chunk, L2p, Dp, wf, Np, dq_acc, dk,
                        dv, prm.part_kv, k, v, st);
    if (s) return s;
  } else {
    auto kern = fold ? tree_attn_bwd_sm100<true> : tree_attn_bwd_sm100<false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
    if (e != cudaSuccess) { set_error("sm100_attn_bwd: smem attribute: %s", cudaGetErrorString(e)); return TT_ERR_CUDA; }
    const unsigned grid = (unsigned)pk.n_blk * hkv;
    kern<<<grid, kBwdThreads, kSmemBytes, st>>>(mq, mk, mv, mdo, mdq, prm);
    count_launch();
    if ((s = check_launch("tree_attn_bwd_sm100"))) return s;
  }
  const int64_t n4 = N * hq * d / 4;
  const int nconv = (int)std::min<int64_t>((n4 + 255) / 256, kDqConvBlocks);
  dq_convert_kernel<<<(unsigned)nconv, 256, 0, st>>>(reinterpret_cast<const float4*>(dq_acc),
                                                     reinterpret_cast<uint2*>(dq), n4, sqnorm ? part_q : nullptr, N, hq);
  count_launch();
  if ((s = check_launch("dq_convert_kernel"))) return s;
  if (!sqnorm) return TT_OK;
  sqnorm_final_kernel<<<1, 256, 0, st>>>(part_q, nconv, part_kv, (int)(pk.n_blk * hkv), sqnorm);
  count_launch();
  return check_launch("sqnorm_final_kernel");
}

}  // namespace tt
