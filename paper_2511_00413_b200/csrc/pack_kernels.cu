// pack_kernels.cu — device half of Tree Packing (tt_pack): per-token artifacts and tile metadata.
//
// Kernel 1 (one 128-thread CTA per 128-token block): the block's first token's node comes from the
// host DFS, each token steps forward to its own node, then writes the Fig. 6impl artifacts:
//   pos = depth(u) + (i - start(u))   (restored position id)
//   w   = leaves(u)                   (tree-scale)
//   E   = sub_end(u)                  (shared-prefix mask as a subtree interval)
//   node = u
// and reduces min / max E over the block's keys.  16 B/token written, coalesced.
// Kernel 2 (one warp per q-block): classifies the tiles (qb, kb <= qb) from minE/maxE and
// compacts the non-empty ones into the triangular fwd list (no global scan needed).  The scan starts
// at kb_lo[qb], the first block of the tree holding the q-block's first token (host-computed): in a
// forest no earlier tree's key is visible, so a batch of trees packs in O(sum of per-tree blocks^2)
// instead of O(total blocks^2).
#include "tt_internal.cuh"

namespace tt {

__global__ void __launch_bounds__(kBlock) pack_fill_kernel(int64_t N, const int32_t* __restrict__ order,
                                                           const int32_t* __restrict__ order_start, int32_t n_order,
                                                           const int32_t* __restrict__ blk_first,
                                                           const int32_t* __restrict__ node_start,
                                                           const int32_t* __restrict__ node_sub_end,
                                                           const int32_t* __restrict__ node_depth,
                                                           const int32_t* __restrict__ node_leaves,
                                                           int32_t* __restrict__ pos, int32_t* __restrict__ w,
                                                           int32_t* __restrict__ E, int32_t* __restrict__ node,
                                                           int32_t* __restrict__ kminE, int32_t* __restrict__ kmaxE) {
  const int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x;
  int32_t e_min = INT32_MAX, e_max = INT32_MIN;
  // the host gives each block the packed-order index of the node holding its first token (nodes with
  // tokens are contiguous and sorted); each thread steps forward over the few nodes the block's 128
  // tokens span
  if (i < N) {
    int32_t lo = __ldg(blk_first + blockIdx.x);
    int steps = 0;
    while (lo + 1 < n_order && order_start[lo + 1] <= i && steps < 8) { ++lo; ++steps; }
    if (steps == 8) {  // many short nodes in this block: binary search the rest of the range
      int32_t hi = min(n_order - 1, lo + kBlock);
      while (lo < hi) {
        int32_t mid = (lo + hi + 1) >> 1;
        if (order_start[mid] <= i) lo = mid; else hi = mid - 1;
      }
    }
    const int32_t u = order[lo];
    const int32_t s = node_start[u];
    const int32_t e = node_sub_end[u];
    pos[i] = node_depth[u] + (int32_t)(i - s);
    w[i] = node_leaves[u];
    E[i] = e;
    node[i] = u;
    e_min = e_max = e;
  }
  // block min / max of E
  for (int off = 16; off > 0; off >>= 1) {
    e_min = min(e_min, __shfl_xor_sync(0xffffffffu, e_min, off));
    e_max = max(e_max, __shfl_xor_sync(0xffffffffu, e_max, off));
  }
  __shared__ int32_t smin[kBlock / 32], smax[kBlock / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { smin[warp] = e_min; smax[warp] = e_max; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < kBlock / 32; ++k) { e_min = min(e_min, smin[k]); e_max = max(e_max, smax[k]); }
    kminE[blockIdx.x] = e_min;
    kmaxE[blockIdx.x] = e_max;
  }
}

__global__ void __launch_bounds__(32) pack_tiles_kernel(int64_t N, int32_t nb, const int32_t* __restrict__ kb_lo,
                                                        const int32_t* __restrict__ kminE,
                                                        const int32_t* __restrict__ kmaxE, int32_t* __restrict__ fwd_cnt,
                                                        int32_t* __restrict__ fwd_list) {
  const int32_t qb = blockIdx.x;
  const int lane = threadIdx.x;
  const int64_t i0 = (int64_t)qb * kBlock;
  const int64_t i1 = imin64(N, i0 + kBlock);
  int32_t* out = fwd_list + tri_off(qb);
  int32_t cnt = 0;
  // 4 x 32 k-blocks per pass: all 8 loads of a pass are issued before the first ballot
  for (int32_t base = kb_lo[qb]; base <= qb; base += 128) {
    int32_t mx[4], mn[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int32_t kb = base + 32 * u + lane;
      mx[u] = kb < qb ? __ldg(kmaxE + kb) : 0;
      mn[u] = kb < qb ? __ldg(kminE + kb) : 0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int32_t kb = base + 32 * u + lane;
      int cls = 0;
      if (kb < qb) cls = (mx[u] <= i0) ? 0 : ((mn[u] >= i1) ? kClsFull : kClsPartial);
      else if (kb == qb) cls = (i1 - i0 == 1) ? kClsFull : kClsPartial;
      const unsigned bal = __ballot_sync(0xffffffffu, cls != 0);
      if (cls != 0) {
        const int slot = cnt + __popc(bal & ((1u << lane) - 1u));
        out[slot] = kb | (cls << kClsShift);
      }
      cnt += __popc(bal);
    }
  }
  if (lane == 0) fwd_cnt[qb] = cnt;
}

tt_status launch_pack_fill(const tt_packed& pk, const int32_t* order, const int32_t* order_start, int32_t n_order,
                           const int32_t* kb_lo, const int32_t* blk_first,
                           int32_t* pos, int32_t* w, int32_t* E, int32_t* node, int32_t* kminE, int32_t* kmaxE,
                           int32_t* fwd_cnt, int32_t* fwd_list, cudaStream_t st) {
  const int32_t nb = pk.n_blk;
  pack_fill_kernel<<<nb, kBlock, 0, st>>>(pk.n_tokens, order, order_start, n_order, blk_first, pk.node_start, pk.node_sub_end,
                                          pk.node_depth, pk.node_leaves, pos, w, E, node, kminE, kmaxE);
  count_launch();
  tt_status s = check_launch("pack_fill_kernel");
  if (s) return s;
  pack_tiles_kernel<<<nb, 32, 0, st>>>(pk.n_tokens, nb, kb_lo, kminE, kmaxE, fwd_cnt, fwd_list);
  count_launch();
  return check_launch("pack_tiles_kernel");
}

}  // namespace tt
