// attn_sm100_fwd.cu — tree-masked attention forward on sm_100a tensor cores (tcgen05 + TMEM + TMA).
//
// What it computes (Eq. 1, with an explicit softmax scale R1 and the shared-prefix mask
// of P:531-533 in its interval form j <= i < E_j, R2):
//   O_i = sum_j softmax_j(scale q_i.k_j) v_j,   LSE_i = ln sum_j exp(scale q_i.k_j)
//
// Design.  One CTA owns two adjacent 128-row query tiles (q-blocks 2p, 2p+1) of one
// head and walks the UNION of their non-empty k-tiles in ascending order (the pack's tile lists);
// empty tiles are never loaded or multiplied, full tiles run unmasked, partial tiles are masked in
// registers.  K/V tiles are shared by both query tiles, so each TMA'd K/V byte feeds two MMAs.
//   warp 0      TMA producer: Q0/Q1 once, then K/V(+E) tiles into a 2-stage ring (SWIZZLE_128B)
//   warp 1      TMEM allocator (512 columns: S0 | S1 | O0 | O1) and MMA issuer (one thread):
//               S_i = Q_i K^T (SS, M=N=128, K=128) into TMEM, then O_i += P_i V with P_i read from
//               TMEM (TS) — FA4-style order PV_0, S_0', PV_1, S_1'
//   warps 2-17  softmax: 2 query tiles x 2 column halves x 4 warps.  One thread per (row, half):
//               tcgen05.ld 32x32b gives each thread its row (TMEM lane quadrant = warp % 4), so row
//               max / sum are thread-local within a half; the halves exchange maxima through smem.
// Softmax keeps the running max in log2 units and only rescales the O accumulator in TMEM when
// the max grows by more than 2^8 (stale-max trick; exact after the final 1/l).  P (bf16) is
// written back over S in TMEM and consumed by the TS MMA; the epilogue divides by l and stores
// O (bf16) and LSE (fp32, natural log).
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
constexpr int kStages = 2;
constexpr int kFwdThreads = 576;  // 18 warps: producer, MMA, 2 query tiles x 2 column halves x 4 softmax warps
constexpr int kConsumerThreads = kFwdThreads - 32;  // MMA warp + softmax warps: release an item's tile list
constexpr uint32_t kTileBytes = 128 * kD * 2;  // 32 KB: two 16 KB SWIZZLE_128B chunks (d 0-63 | 64-127)
constexpr uint32_t kChunkBytes = 128 * 64 * 2;
constexpr uint32_t kOffQ = 0;                       // Q0, Q1
constexpr uint32_t kOffKV = 2 * kTileBytes;         // stage s: K at +s*64K, V at +s*64K+32K
constexpr uint32_t kOffE = kOffKV + kStages * 2 * kTileBytes;  // E of the stage's 128 keys (512 B)
constexpr uint32_t kOffBar = kOffE + kStages * 512;
// q_full, full[2], empty[2], s_full[2], p_full[2], o_full[2], item_full[2], item_empty[2], q_free, clc
constexpr uint32_t kNumBars = 1 + 2 * kStages + 6 + 4 + 2;
constexpr uint32_t kOffMisc = (kOffBar + kNumBars * 8 + 15) & ~15u;  // [0] TMEM base
constexpr uint32_t kOffInfo = kOffMisc + 16;        // per item buffer: {item, T (-1: no more items), has1, 0}
constexpr uint32_t kOffClc = kOffInfo + 2 * 16;     // cluster-launch-control response (16 B)
constexpr uint32_t kOffX = kOffClc + 16;            // row-max exchange [2 parity][2 tiles][2 halves][128] + l [2][2][128]
constexpr uint32_t kOffTiles = kOffX + (2 * 2 * 2 * 128 + 2 * 2 * 128) * 4;
constexpr float kRescaleThreshold = 8.0f;  // log2 units
// the next item is claimed (CLC) when the producer loads the current item's k-tile T - kClaimAhead and
// its tile list built from k-tile T - kPrepareAhead on
#ifndef TT_FWD_CLAIM_AHEAD
#define TT_FWD_CLAIM_AHEAD 5
#endif
#ifndef TT_FWD_PREPARE_AHEAD
#define TT_FWD_PREPARE_AHEAD 3
#endif
constexpr int kClaimAhead = TT_FWD_CLAIM_AHEAD, kPrepareAhead = TT_FWD_PREPARE_AHEAD;

__device__ unsigned long long g_fwd_dbg[16];  // development instrumentation (TT_DEBUG_FWD & 8)

struct FwdParams {
  int64_t N;
  int hq, hkv, nb, npairs;
  float scale_log2;
  int chunk;  // CTA order: query-block pairs (heaviest first) in chunks of `chunk`; within a chunk the kv
              // heads outermost (1 = heads fastest, >= npairs = head-major: K/V of one group L2-resident)
  int steal;  // persistent CTAs: take over not-yet-launched CTAs' items (dev A/B TT_FWD_NOSTEAL: 0)
  int dbg;
  int wait;  // dev A/B (TT_WAIT_HINT): suspend-hint waits, bit 0 producer, 1 softmax, 2 epilogue
  const int32_t* E;
  const int32_t* fwd_cnt;
  const int32_t* fwd_list;
  __nv_bfloat16* o;
  float* lse;
};

__device__ __forceinline__ int tile_cls(int32_t e, int i) { return (e >> (28 + 2 * i)) & 3; }

// work item x (a blockIdx.x of the grid) -> (query-block pair, q head): heavy (late) query blocks first,
// the q heads of one kv head adjacent, in chunks of p.chunk pairs
__device__ __forceinline__ void fwd_item(const FwdParams& p, int x, int& pair, int& h) {
  const int gq = p.hq / p.hkv;
  const int per = p.chunk * p.hq;
  const int ch = x / per, w = x - ch * per;
  const int len = min(p.chunk, p.npairs - ch * p.chunk);
  const int hkk = w / (len * gq), w2 = w - hkk * (len * gq);
  pair = p.npairs - 1 - (ch * p.chunk + w2 / gq);
  h = hkk * gq + w2 % gq;
}

// Persistent over work items: the grid has one CTA per (query-block pair, head) and the hardware
// launches them in order (heaviest first), but a running CTA takes over the next not-yet-launched CTA's
// item through cluster launch control (clc_try_cancel) a few tiles before its current item ends, so
// item n+1's Q / first K/V loads, tile list and first S MMAs overlap item n's last tiles and epilogue
// instead of a CTA exit, launch, barrier init and TMEM allocation.  Each item's merged tile list is built by the producer warp
// into one of two buffers (item_full / item_empty hand them to the MMA and softmax warps).
__global__ void __launch_bounds__(kFwdThreads, 1)
    tree_attn_fwd_sm100(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                        const __grid_constant__ CUtensorMap tmV, const FwdParams p) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned base; pointer arithmetic on smem_raw keeps the shared address space visible to
  // the compiler (LDS/STS instead of generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar);
  uint64_t* bar_q = bars;
  uint64_t* full = bars + 1;
  uint64_t* empty = bars + 1 + kStages;
  uint64_t* s_full = bars + 1 + 2 * kStages;
  uint64_t* p_full = s_full + 2;
  uint64_t* o_full = s_full + 4;
  uint64_t* item_full = s_full + 6;   // [2] tile list + info of an item written (32 producer lanes)
  uint64_t* item_empty = s_full + 8;  // [2] item's tile list no longer read (every consumer thread)
  uint64_t* q_free = s_full + 10;     // the item's last S MMAs (the last reads of Q) completed
  uint64_t* clc_bar = s_full + 11;
  uint32_t* misc = reinterpret_cast<uint32_t*>(smem + kOffMisc);
  int4* info = reinterpret_cast<int4*>(smem + kOffInfo);
  const int tl_stride = p.nb + 4;
  int32_t* tiles_buf = reinterpret_cast<int32_t*>(smem + kOffTiles);  // [2][nb + 4]
  uint8_t* flags0 = reinterpret_cast<uint8_t*>(tiles_buf + 2 * tl_stride);
  uint8_t* flags1 = flags0 + p.nb + 4;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long t_kernel0 = TT_CLK();

  if (warp == 1 && lane == 0) {
    mbar_init(bar_q, 1);
    for (int s = 0; s < kStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&s_full[i], 1); mbar_init(&p_full[i], 256); mbar_init(&o_full[i], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&item_full[b], 32); mbar_init(&item_empty[b], kConsumerThreads); }
    mbar_init(q_free, 1);
    mbar_init(clc_bar, 1);
    mbar_fence_init();
  }
  __syncthreads();
  uint32_t tmem = 0;
  if (warp == 1) {
    tmem_alloc(&misc[0], 512);
    tmem_relinquish();
  }
  if (warp != 0) {
    // TMEM base visible to the MMA and softmax warps (the producer never touches TMEM and starts its
    // loads at once); named barrier 5 over warps 1..17
    tc_fence_before();
    named_bar_sync(5, kFwdThreads - 32);
    tc_fence_after();
    tmem = misc[0];
  }

  if (warp == 0) {
    // ===================== producer warp: scheduler, tile lists, TMA =====================
    const int gq = p.hq / p.hkv;
    bool steal = p.steal != 0;
    uint32_t clc_ph = 0;
    if (lane == 0) {
      tma_prefetch(&tmQ);
      tma_prefetch(&tmK);
      tma_prefetch(&tmV);
    }
    auto has1_of = [&](int qa) { return qa + 1 < p.nb && !(dev_dbg(p.dbg) & 16); };  // dbg 16: drop query tile 1
    // merged tile list of an item's two query blocks (kb | cls0 << 28 | cls1 << 30, ascending) into
    // buffer b, published with info[b] = {item, T, last tile of query tile 0, last tile of query tile 1}
    auto build_list = [&](int b, int x, int qa, bool has1) -> int {
      const int kb_end = has1 ? qa + 2 : qa + 1;
      for (int k = lane; k < kb_end; k += 32) { flags0[k] = 0; flags1[k] = 0; }
      __syncwarp();
      auto fill = [&](uint8_t* fl, int qb) {
        const int n = p.fwd_cnt[qb];
        const int32_t* l = p.fwd_list + tri_off(qb);
        for (int k0 = 0; k0 < n; k0 += 128) {  // 4 independent loads in flight per lane
          int32_t v[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) v[u] = (k0 + 32 * u + lane < n) ? l[k0 + 32 * u + lane] : -1;
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (v[u] >= 0) fl[v[u] & kKbMask] = (uint8_t)(v[u] >> kClsShift);
        }
      };
      fill(flags0, qa);
      if (has1) fill(flags1, qa + 1);
      __syncwarp();
      int32_t* tl = tiles_buf + b * tl_stride;
      int cnt = 0, last0 = -1, last1 = -1;
      for (int base = 0; base < kb_end; base += 32) {
        const int kb = base + lane;
        const int v = kb < kb_end ? (flags0[kb] | (flags1[kb] << 2)) : 0;
        const unsigned bal = __ballot_sync(0xffffffffu, v != 0);
        const unsigned b0 = __ballot_sync(0xffffffffu, (v & 3) != 0);
        const unsigned b1 = __ballot_sync(0xffffffffu, (v >> 2) != 0);
        if (v) tl[cnt + __popc(bal & ((1u << lane) - 1u))] = kb | (v << kClsShift);
        if (b0) last0 = cnt + __popc(bal & (uint32_t)((2ull << (31 - __clz(b0))) - 1ull)) - 1;
        if (b1) last1 = cnt + __popc(bal & (uint32_t)((2ull << (31 - __clz(b1))) - 1ull)) - 1;
        cnt += __popc(bal);
      }
      if (lane == 0) info[b] = make_int4(x, cnt, last0, last1);
      mbar_arrive(&item_full[b]);  // every lane: releases its own list writes
      return cnt;
    };
    auto load_q = [&](int qa, bool has1, int hh) {
      mbar_expect_tx(bar_q, (has1 ? 2 : 1) * kTileBytes);
      for (int i = 0; i < (has1 ? 2 : 1); ++i)
        for (int c = 0; c < 2; ++c)
          tma_load_3d(smem + kOffQ + i * kTileBytes + c * kChunkBytes, &tmQ, bar_q, c * 64, hh, (qa + i) * 128);
    };
    auto load_kv = [&](uint32_t g, int kb, int hh) {
      const int s = (int)(g % kStages);
      uint8_t* kd = smem + kOffKV + s * 2 * kTileBytes;
      const int hk = hh / gq;
      mbar_expect_tx(&full[s], 2 * kTileBytes + 512);
      bulk_load_1d(smem + kOffE + s * 512, p.E + (int64_t)kb * 128, 512, &full[s]);
      for (int c = 0; c < 2; ++c) tma_load_3d(kd + c * kChunkBytes, &tmK, &full[s], c * 64, hk, kb * 128);
      for (int c = 0; c < 2; ++c) tma_load_3d(kd + kTileBytes + c * kChunkBytes, &tmV, &full[s], c * 64, hk, kb * 128);
    };
    // item 0: Q and its first K/V tile go out before the tile-list merge (the first merged k-tile is
    // the smaller of the two lists' first entries: both ascending)
    int x = (int)blockIdx.x, pair, h;
    fwd_item(p, x, pair, h);
    int qa = 2 * pair;
    bool has1 = has1_of(qa);
    if (lane == 0) {
      load_q(qa, has1, h);
      int kb0 = p.fwd_list[tri_off(qa)] & kKbMask;
      if (has1) kb0 = min(kb0, p.fwd_list[tri_off(qa + 1)] & kKbMask);
      load_kv(0, kb0, h);
    }
    int T = build_list(0, x, qa, has1);
    uint32_t g = 1;  // k-tiles issued so far (all items): stage g % kStages
    int t_first = 1;
    for (int n = 0;; ++n) {
      const int b = n & 1;
      const int32_t* tl = tiles_buf + b * tl_stride;
      // The next item (through the CLC) is prepared while this item's last k-tiles are loaded (the
      // producer runs ~2 tiles ahead of the MMAs), so its tile list is ready when this item's MMAs end.
      // (claimed late, a few tiles before this item's end: claiming at an item's start would pair heavy
      // items on one CTA and unbalance the tail)
      int xn = -1, pair_n = 0, h_n = 0, T_n = 0;
      bool has1_n = false, claimed = false, prepared = false;
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
          xn = clc_query_x(smem + kOffClc);
          fence_proxy_async_smem();
          __syncwarp();
          if (xn < 0) steal = false;  // no further request after a failed one
        }
        if (n >= 1) mbar_wait(&item_empty[b ^ 1], ((n - 1) >> 1) & 1);  // item n-1 released buffer b^1
        if (xn < 0) {
          if (lane == 0) info[b ^ 1] = make_int4(-1, -1, -1, -1);
          mbar_arrive(&item_full[b ^ 1]);
          return;
        }
        fwd_item(p, xn, pair_n, h_n);
        has1_n = has1_of(2 * pair_n);
        T_n = build_list(b ^ 1, xn, 2 * pair_n, has1_n);
      };
      for (int t = t_first; t < T; ++t, ++g) {
        const int s = (int)(g % kStages);
        if (g >= (uint32_t)kStages) mbar_wait_role(&empty[s], ((g / kStages) - 1) & 1, dev_dbg(p.wait) & 1);
        if (lane == 0) load_kv(g, tl[t] & kKbMask, h);
        if (!claimed && t >= T - kClaimAhead) claim();
        if (!prepared && t >= T - kPrepareAhead) prepare_next();
      }
      if (!prepared) prepare_next();
      if (xn < 0) break;
      x = xn;
      pair = pair_n;
      h = h_n;
      qa = 2 * pair;
      has1 = has1_n;
      T = T_n;
      mbar_wait(q_free, n & 1);  // item n's last S MMAs have read Q
      if (lane == 0) load_q(qa, has1, h);
      t_first = 0;
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (whole warp converged, one elected lane issues) ==========
    constexpr uint32_t idS = idesc_bf16(128, 128, 0, 0);  // Q (K-major) x K^T (K-major)
    constexpr uint32_t idO = idesc_bf16(128, 128, 0, 1);  // P (TMEM, K-major) x V (MN-major)
    const uint32_t qbase = warp_uniform(smem_u32(smem + kOffQ));
    const uint32_t tm = warp_uniform(tmem);
    uint32_t g = 0;  // k-tiles consumed so far (all items)
    uint32_t pph[2] = {0, 0};
    long long w_p = 0, w_kv = 0, w_item = 0, t_beg = TT_CLK();
    int n_items = 0;
    for (int n = 0;; ++n) {
      const int b = n & 1;
      const long long t_item = TT_CLK();  // item boundary: from here to the item's first S issue
      mbar_wait(&item_full[b], (n >> 1) & 1);
      const int4 inf = info[b];
      const int T = inf.y;
      if (T < 0) break;
      const int32_t* tiles = tiles_buf + b * tl_stride;
      auto issue_S = [&](int i, int t) {
        const uint32_t kbase = qbase + kOffKV + ((g + t) % kStages) * 2 * kTileBytes;
        const uint32_t qb = qbase + i * kTileBytes;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = (kk >> 2) * kChunkBytes + (kk & 3) * 32;
          mma_ss_w(tm + 128 * i, sdesc(qb + off, 16, 1024), sdesc(kbase + off, 16, 1024), idS, kk > 0);
        }
        mma_commit_w(&s_full[i]);
      };
      const int last[2] = {inf.z, inf.w};  // each query tile's last k-tile (the producer's list build)
      bool first[2] = {true, true};
      mbar_wait(bar_q, n & 1);
      if (T > 0) {
        mbar_wait(&full[g % kStages], (g / kStages) & 1);
        if ((dev_dbg(p.dbg) & 8) && lane == 0 && n == 0) atomicAdd(&g_fwd_dbg[8], (unsigned long long)(TT_CLK() - t_kernel0));
        tc_fence_after();
#pragma unroll
        for (int i = 0; i < 2; ++i)
          if (tile_cls(tiles[0], i)) issue_S(i, 0);
      }
      if (n > 0) w_item += TT_CLK() - t_item;
      ++n_items;
      if (T <= 1) mma_commit_w(q_free);
      for (int t = 0; t < T; ++t) {
        const uint32_t s = (g + t) % kStages;
        const uint32_t vbase = qbase + kOffKV + s * 2 * kTileBytes + kTileBytes;
        bool waited = false;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          if (tile_cls(tiles[t], i)) {
            { long long t0 = TT_CLK(); mbar_wait(&p_full[i], pph[i]); w_p += TT_CLK() - t0; }
            pph[i] ^= 1;
            tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
              // P of keys [16 kk, 16 kk + 16): packed by column half kk / 4 at S column 64 (kk / 4) + 8 (kk % 4)
              mma_ts_w(tm + 256 + 128 * i, tm + 128 * i + 8 * kk + ((kk >> 2) << 5), sdesc(vbase + kk * 2048, kChunkBytes, 1024), idO,
                       (!first[i] || kk > 0) ? 1u : 0u);
            first[i] = false;
            if (t == last[i]) mma_commit_w(&o_full[i]);
          }
          if (t + 1 < T && tile_cls(tiles[t + 1], i)) {
            if (!waited) {
              { long long t0 = TT_CLK(); mbar_wait(&full[(g + t + 1) % kStages], ((g + t + 1) / kStages) & 1); w_kv += TT_CLK() - t0; }
              tc_fence_after();
              waited = true;
            }
            issue_S(i, t + 1);
          }
        }
        if (t + 2 == T) mma_commit_w(q_free);  // the item's last S MMAs were issued just above
        mma_commit_w(&empty[s]);
      }
      g += (uint32_t)T;
      mbar_arrive(&item_empty[b]);
    }
    if ((dev_dbg(p.dbg) & 8) && lane == 0) {
      atomicAdd(&g_fwd_dbg[0], (unsigned long long)(TT_CLK() - t_beg));
      atomicAdd(&g_fwd_dbg[1], (unsigned long long)w_p);
      atomicAdd(&g_fwd_dbg[2], (unsigned long long)w_kv);
      atomicAdd(&g_fwd_dbg[3], (unsigned long long)g);
      atomicAdd(&g_fwd_dbg[14], (unsigned long long)w_item);
      atomicAdd(&g_fwd_dbg[15], (unsigned long long)n_items);
    }
  } else {
    // ===================== softmax: 2 query tiles x 2 column halves =====================
    // Warpgroup (i, hf) owns rows of query tile i (one thread per row: its TMEM lane) and key columns
    // [64 hf, 64 hf + 64) of every k-tile.  The two halves exchange their row maxima through shared
    // memory (one named barrier per tile), keep separate partial row sums (same running max), rescale
    // their own half of O, and pack P (bf16) over their OWN S columns so neither half can overwrite
    // scores the other has not read yet.
    const int i = (warp - 2) >> 3;           // query tile
    const int hf = ((warp - 2) >> 2) & 1;    // column half
    const int q = warp & 3;                  // TMEM lane quadrant
    const int r = q * 32 + lane;
    const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
    const uint32_t tSh = tl + 128 * i + 64 * hf;        // this half's S columns (P packed at [tSh, tSh + 32))
    const uint32_t tOh = tl + 256 + 128 * i + 64 * hf;  // this half's O columns
    float* xmax = reinterpret_cast<float*>(smem + kOffX);  // [parity][tile][half][row]
    float* xl = xmax + 2 * 2 * 2 * 128;                    // [tile][half][row]
    const float sl2 = p.scale_log2;
    uint32_t sph = 0, par = 0, oph = 0, g = 0;
    long long c_ws = 0, c_cmp = 0, c_n = 0, c_bar = 0, c_ldp = 0, c_mx = 0, c_ex = 0;
    for (int n = 0;; ++n) {
      const int b = n & 1;
      mbar_wait(&item_full[b], (n >> 1) & 1);
      const int4 inf = info[b];
      const int T = inf.y;
      if (T < 0) break;
      const int32_t* tiles = tiles_buf + b * tl_stride;
      int pair, h;
      fwd_item(p, inf.x, pair, h);
      const int64_t row = (int64_t)(2 * pair + i) * 128 + r;
      if (i == 0 || inf.w >= 0) {  // query tile 1 exists
        float m = -INFINITY, l = 0.f;
        bool first = true;
        for (int t = 0; t < T; ++t) {
          const int32_t e = tiles[t];
          const int cls = tile_cls(e, i);
          if (!cls) continue;
          const int kb = e & kKbMask;
          const int64_t j0 = (int64_t)kb * 128 + 64 * hf;  // first key of this half
          { const long long t0 = TT_CLK(); mbar_wait_role(&s_full[i], sph, dev_dbg(p.wait) & 2); c_ws += TT_CLK() - t0; }
          const long long t_cmp = TT_CLK();
          sph ^= 1;
          tc_fence_after();
          if (dev_dbg(p.dbg) & 32) {  // development ablation: no softmax work (MMA pipeline alone)
            tc_fence_before();
            mbar_arrive(&p_full[i]);
            continue;
          }
          uint32_t s[64];
          tmem_ld32(tSh, *reinterpret_cast<uint32_t(*)[32]>(&s[0]));
          tmem_ld32(tSh + 32, *reinterpret_cast<uint32_t(*)[32]>(&s[32]));
          tmem_wait_ld();
          c_ldp += TT_CLK() - t_cmp;
          // ---- mask (partial tiles; key columns past N on the ragged last block) ----
          const bool ragged = j0 + 64 > p.N;
          if (cls == kClsPartial && !(dev_dbg(p.dbg) & 64)) {  // dbg 64: development ablation, partial tiles unmasked
            // int32 index math (N < 2^31): key c allowed iff c <= row - j0, c < N - j0, row < E_c
            const int4* Es = reinterpret_cast<const int4*>(smem + kOffE + ((g + t) % kStages) * 512) + 16 * hf;
            const int irow = (int)row;
            if (kb != (int)(row >> 7) && !(dev_dbg(p.dbg) & 128)) {  // dbg 128: dev A/B, full test everywhere
              // below the diagonal (kb < query block) every key precedes every row and no key is past N:
              // only the subtree-end test (warp-uniform branch)
#pragma unroll
              for (int c4 = 0; c4 < 16; ++c4) {
                const int4 ev = Es[c4];
                const int ee[4] = {ev.x, ev.y, ev.z, ev.w};
#pragma unroll
                for (int u = 0; u < 4; ++u)
                  if (irow >= ee[u]) s[4 * c4 + u] = __float_as_uint(-INFINITY);
              }
            } else {
              const int cmax = min((int)(row - j0), (int)(p.N - j0) - 1);
#pragma unroll
              for (int c4 = 0; c4 < 16; ++c4) {
                const int4 ev = Es[c4];
                const int ee[4] = {ev.x, ev.y, ev.z, ev.w};
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                  const int c = 4 * c4 + u;
                  if (!((c <= cmax) && (irow < ee[u]))) s[c] = __float_as_uint(-INFINITY);
                }
              }
            }
          } else if (ragged) {
            const int jmax = (int)(p.N - j0);
#pragma unroll
            for (int c = 0; c < 64; ++c)
              if (c >= jmax) s[c] = __float_as_uint(-INFINITY);
          }
          // ---- row max: 4 partial maxima, exchange with the other half ----
          float pm[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) pm[u] = __uint_as_float(s[u]);
#pragma unroll
          for (int c = 4; c < 64; c += 4)
#pragma unroll
            for (int u = 0; u < 4; ++u) pm[u] = fmaxf(pm[u], __uint_as_float(s[c + u]));
          const float hmax = fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3]));
          c_mx += TT_CLK() - t_cmp;
          xmax[((par * 2 + i) * 2 + hf) * 128 + r] = hmax;
          { const long long tb = TT_CLK(); named_bar_sync(1 + i, 256); c_bar += TT_CLK() - tb; }
          const float mx = fmaxf(hmax, xmax[((par * 2 + i) * 2 + (hf ^ 1)) * 128 + r]);
          par ^= 1;
          const float m_new = fmaxf(m, mx * sl2);
          const bool resc = (m == -INFINITY) ? (m_new != -INFINITY) : (m_new > m + kRescaleThreshold);
          const float m_use = resc ? m_new : m;
          const float corr = (m == -INFINITY) ? 0.f : ex2(m - m_use);
          const float mb = (m_use == -INFINITY) ? 0.f : m_use;
          // ---- P = exp2(s * scale_log2 - m): packed f32x2 FMAs; on unmasked tiles a quarter of the
          //      exponentials run as a polynomial on the FMA pipe (FA4-style) ----
          const float2 SL = make_float2(sl2, sl2), NM = make_float2(-mb, -mb);
          float2 acc0 = make_float2(0.f, 0.f), acc1 = make_float2(0.f, 0.f);
          if ((cls == kClsFull || (dev_dbg(p.dbg) & 64)) && !ragged) {
#pragma unroll
            for (int c = 0; c < 64; c += 4) {
              const float2 a01 = ffma2(make_float2(__uint_as_float(s[c]), __uint_as_float(s[c + 1])), SL, NM);
              const float2 a23 = ffma2(make_float2(__uint_as_float(s[c + 2]), __uint_as_float(s[c + 3])), SL, NM);
              const float2 p01 = make_float2(ex2(a01.x), ex2(a01.y));
#ifndef TT_FWD_POLY
#define TT_FWD_POLY 1
#endif
              // 2 x TT_FWD_POLY of every 8 exponentials run on the FMA pipe (measured best: 1, i.e. 25%;
              // the polynomial costs ~8 FMA-pipe cycles per element vs 8 MUFU cycles per exp)
              const float2 p23 = (TT_FWD_POLY == 2 || (TT_FWD_POLY == 1 && (c & 4))) ? exp2_poly2(a23)
                                                                                     : make_float2(ex2(a23.x), ex2(a23.y));
              acc0 = fadd2(acc0, p01);
              acc1 = fadd2(acc1, p23);
              s[c >> 1] = pack_bf16(p01.x, p01.y);
              s[(c >> 1) + 1] = pack_bf16(p23.x, p23.y);
            }
          } else {
            // masked / ragged tiles: masked scores are -inf; the polynomial share uses the variant that
            // returns exactly 0 there
#pragma unroll
            for (int c = 0; c < 64; c += 4) {
              const float2 a01 = ffma2(make_float2(__uint_as_float(s[c]), __uint_as_float(s[c + 1])), SL, NM);
              const float2 a23 = ffma2(make_float2(__uint_as_float(s[c + 2]), __uint_as_float(s[c + 3])), SL, NM);
              const float2 p01 = make_float2(ex2(a01.x), ex2(a01.y));
              const float2 p23 = (TT_FWD_POLY == 2 || (TT_FWD_POLY == 1 && (c & 4))) ? exp2_poly2z(a23)
                                                                                     : make_float2(ex2(a23.x), ex2(a23.y));
              acc0 = fadd2(acc0, p01);
              acc1 = fadd2(acc1, p23);
              s[c >> 1] = pack_bf16(p01.x, p01.y);
              s[(c >> 1) + 1] = pack_bf16(p23.x, p23.y);
            }
          }
          c_ex += TT_CLK() - t_cmp;
          const float2 accs = fadd2(acc0, acc1);
          l = l * corr + (accs.x + accs.y);
          m = m_use;
          // ---- lazy rescale of this half of O (PV of the previous tile has completed: its commit
          //      precedes the s_full arrival we waited on) ----
          if (!first && __any_sync(0xffffffffu, resc)) {
#pragma unroll 1
            for (int cc = 0; cc < 2; ++cc) {
              uint32_t ov[32];
              tmem_ld32(tOh + 32 * cc, ov);
              tmem_wait_ld();
#pragma unroll
              for (int u = 0; u < 32; ++u) ov[u] = __float_as_uint(__uint_as_float(ov[u]) * corr);
              tmem_st32(tOh + 32 * cc, ov);
            }
          }
          tmem_st32(tSh, *reinterpret_cast<uint32_t(*)[32]>(&s[0]));
          tmem_wait_st();
          tc_fence_before();
          mbar_arrive(&p_full[i]);
          c_cmp += TT_CLK() - t_cmp;
          ++c_n;
          first = false;
        }
        // ---- epilogue: O / l -> bf16 (this half's 64 columns), LSE (half 0).  The O columns are free
        //      for the next item's first PV once these tcgen05.ld completed: that PV waits for the next
        //      item's first p_full, which these threads arrive on only after this epilogue ----
        mbar_wait_role(&o_full[i], oph, dev_dbg(p.wait) & 4);
        oph ^= 1;
        tc_fence_after();
        xl[(i * 2 + hf) * 128 + r] = l;
        named_bar_sync(1 + i, 256);
        const float lt = xl[(i * 2) * 128 + r] + xl[(i * 2 + 1) * 128 + r];
        const float inv = (lt > 0.f) ? 1.f / lt : 0.f;
        __nv_bfloat16* orow = p.o + (row * p.hq + h) * kD + 64 * hf;
#pragma unroll 1
        for (int cc = 0; cc < 2; ++cc) {
          uint32_t ov[32];
          tmem_ld32(tOh + 32 * cc, ov);
          tmem_wait_ld();
          if (row < p.N) {
            uint32_t pk[16];
#pragma unroll
            for (int u = 0; u < 16; ++u)
              pk[u] = pack_bf16(__uint_as_float(ov[2 * u]) * inv, __uint_as_float(ov[2 * u + 1]) * inv);
            uint4* dst = reinterpret_cast<uint4*>(orow + 32 * cc);
#pragma unroll
            for (int u = 0; u < 4; ++u) dst[u] = make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
          }
        }
        if (hf == 0 && row < p.N) p.lse[(int64_t)h * p.N + row] = (m + __log2f(lt)) * kLn2;
      }
      g += (uint32_t)T;
      mbar_arrive(&item_empty[b]);
    }
    if ((dev_dbg(p.dbg) & 8) && r == 0 && i == 0 && hf == 0) {
      atomicAdd(&g_fwd_dbg[4], (unsigned long long)c_ws);
      atomicAdd(&g_fwd_dbg[5], (unsigned long long)c_cmp);
      atomicAdd(&g_fwd_dbg[6], (unsigned long long)c_n);
      atomicAdd(&g_fwd_dbg[7], (unsigned long long)c_bar);
      atomicAdd(&g_fwd_dbg[9], (unsigned long long)c_ldp);
      atomicAdd(&g_fwd_dbg[10], (unsigned long long)c_mx);
      atomicAdd(&g_fwd_dbg[11], (unsigned long long)c_ex);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
  if ((dev_dbg(p.dbg) & 8) && threadIdx.x == 0) {
    atomicAdd(&g_fwd_dbg[12], (unsigned long long)(TT_CLK() - t_kernel0));
    atomicAdd(&g_fwd_dbg[13], 1ull);
  }
}

}  // namespace

// ------------------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

// [rows, heads, d] bf16 ("thd") as a 3-D tensor map with a {64, 1, box_rows} SWIZZLE_128B box.
tt_status make_tmap_thd(CUtensorMap* m, const void* ptr, int64_t rows, int heads, int d, int box_rows,
                        CUtensorMapDataType dt, int elem_bytes, CUtensorMapSwizzle sw, int box_inner) {
  auto fn = encode_fn();
  if (!fn) { set_error("cuTensorMapEncodeTiled unavailable"); return TT_ERR_CUDA; }
  cuuint64_t dims[3] = {(cuuint64_t)d, (cuuint64_t)heads, (cuuint64_t)rows};
  cuuint64_t strides[2] = {(cuuint64_t)d * elem_bytes, (cuuint64_t)heads * d * elem_bytes};
  cuuint32_t box[3] = {(cuuint32_t)box_inner, 1, (cuuint32_t)box_rows};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(m, dt, 3, const_cast<void*>(ptr), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { set_error("cuTensorMapEncodeTiled failed (%d)", (int)r); return TT_ERR_CUDA; }
  return TT_OK;
}

// generic 3-D tensor map (dims / strides in elements of elem_bytes, innermost first), no swizzle
tt_status make_tmap_3d(CUtensorMap* m, const void* ptr, CUtensorMapDataType dt, int elem_bytes, const int64_t dims3[3],
                       const int64_t strides2[2], const int box3[3]) {
  auto fn = encode_fn();
  if (!fn) { set_error("cuTensorMapEncodeTiled unavailable"); return TT_ERR_CUDA; }
  cuuint64_t dims[3] = {(cuuint64_t)dims3[0], (cuuint64_t)dims3[1], (cuuint64_t)dims3[2]};
  cuuint64_t strides[2] = {(cuuint64_t)strides2[0] * elem_bytes, (cuuint64_t)strides2[1] * elem_bytes};
  cuuint32_t box[3] = {(cuuint32_t)box3[0], (cuuint32_t)box3[1], (cuuint32_t)box3[2]};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(m, dt, 3, const_cast<void*>(ptr), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { set_error("cuTensorMapEncodeTiled failed (%d)", (int)r); return TT_ERR_CUDA; }
  return TT_OK;
}

extern "C" int tt_debug_fwd_counters(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, g_fwd_dbg, sizeof(g_fwd_dbg));
  if (reset) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(g_fwd_dbg, z, sizeof(z));
  }
  return 0;
}

size_t sm100_fwd_smem_bytes(int nb) {
  return 1024 + kOffTiles + 2 * (size_t)(nb + 4) * 4 + 2 * (size_t)(nb + 4) + 16;
}

tt_status sm100_attn_fwd(const tt_packed& pk, const void* q, const void* k, const void* v, int hq, int hkv, int d,
                         float scale, void* o, float* lse, cudaStream_t st) {
  if (d != kD) { set_error("sm100_attn_fwd: d must be 128"); return TT_ERR_UNSUPPORTED; }
  const int nb = pk.n_blk;
  const size_t smem = sm100_fwd_smem_bytes(nb);
  if (smem > 232448) { set_error("sm100_attn_fwd: %d blocks exceed the tile-list smem budget", nb); return TT_ERR_TOO_LARGE; }
  CUtensorMap mq, mk, mv;
  tt_status s;
  if ((s = make_tmap_thd(&mq, q, pk.n_tokens, hq, d, 128, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, CU_TENSOR_MAP_SWIZZLE_128B, 64))) return s;
  if ((s = make_tmap_thd(&mk, k, pk.n_tokens, hkv, d, 128, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, CU_TENSOR_MAP_SWIZZLE_128B, 64))) return s;
  if ((s = make_tmap_thd(&mv, v, pk.n_tokens, hkv, d, 128, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, CU_TENSOR_MAP_SWIZZLE_128B, 64))) return s;
  FwdParams prm;
  prm.N = pk.n_tokens;
  prm.hq = hq;
  prm.hkv = hkv;
  prm.nb = nb;
  prm.npairs = (nb + 1) / 2;
  prm.scale_log2 = scale * kLog2e;
  {
    const char* e = dev_getenv("TT_DEBUG_FWD");
    prm.dbg = e ? atoi(e) : 0;
    const char* o = dev_getenv("TT_CTA_ORDER");  // development A/B: bit 0 = fwd head-major
    prm.chunk = fwd_cta_chunk(pk, prm.npairs, hkv);
    if (o && (atoi(o) & 1)) prm.chunk = prm.npairs;  // development A/B: head-major
    if (const char* c = dev_getenv("TT_FWD_CHUNK")) prm.chunk = atoi(c) > 0 ? atoi(c) : 1;
    const char* wh = dev_getenv("TT_WAIT_HINT");
    prm.wait = wh ? atoi(wh) : 0;
    prm.steal = dev_getenv("TT_FWD_NOSTEAL") ? 0 : 1;  // development A/B: one item per CTA
  }
  prm.E = pk.E;
  prm.fwd_cnt = pk.fwd_cnt;
  prm.fwd_list = pk.fwd_list;
  prm.o = static_cast<__nv_bfloat16*>(o);
  prm.lse = lse;
  cudaError_t e = cudaFuncSetAttribute(tree_attn_fwd_sm100, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) { set_error("sm100_attn_fwd: smem attribute: %s", cudaGetErrorString(e)); return TT_ERR_CUDA; }
  const unsigned grid = (unsigned)prm.npairs * hq;
  tree_attn_fwd_sm100<<<grid, kFwdThreads, smem, st>>>(mq, mk, mv, prm);
  count_launch();
  return check_launch("tree_attn_fwd_sm100");
}

}  // namespace tt
