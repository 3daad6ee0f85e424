// tt_api.cu — C ABI entry points of libtt.so: argument validation, the O(n_nodes) host part of
// Tree Packing, workspace carving and kernel dispatch.  See include/tt.h for the contract.
#include <cmath>
#include <algorithm>
#include <cstring>
#include <vector>

#include "tt_internal.cuh"

namespace tt {

static thread_local std::string g_err;
static thread_local int64_t g_launches = 0;

void set_error(const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
}
void clear_error() { g_err.clear(); }
void count_launch(int n) { g_launches += n; }

tt_status check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return TT_ERR_CUDA;
  }
  return TT_OK;
}

// ------------------------------------------------------------------------------------------
// Host part of Tree Packing: validate, iterative DFS pre-order (roots ascending, children
// ascending; R3), subtree ends, leaf counts (tree-scale) and continuation lists.
// ------------------------------------------------------------------------------------------
struct HostPack {
  int32_t n = 0;
  int64_t N = 0;
  std::vector<int32_t> start, len, sub_end, depth, leaves;  // per node
  std::vector<int32_t> root_start;                          // per node: first token of its tree
  std::vector<int32_t> succ_ptr, succ_tok;                  // per node CSR
  std::vector<int32_t> order, order_start;                  // nodes with len > 0, packed order
  std::vector<int32_t> pre, kids_ptr, kids;                 // DFS pre-order, children CSR
  int32_t n_roots = 0;
  int64_t n_traj = 0, lin_tokens = 0, pairs = 0, lin_pairs = 0;
};

static tt_status host_pack(const int32_t* parent, const int32_t* len, const int32_t* term, int32_t n, HostPack& H) {
  if (!parent || !len) { set_error("tt_pack: parent/len must be non-null host pointers"); return TT_ERR_INVALID_ARGUMENT; }
  if (n <= 0) { set_error("tt_pack: n_nodes must be > 0 (got %d)", n); return TT_ERR_INVALID_ARGUMENT; }
  H.n = n;
  std::vector<int32_t> child_cnt(n + 1, 0);
  int64_t total = 0;
  for (int32_t v = 0; v < n; ++v) {
    if (len[v] < 0) { set_error("tt_pack: len[%d] = %d < 0", v, len[v]); return TT_ERR_INVALID_ARGUMENT; }
    if (term && term[v] < 0) { set_error("tt_pack: term[%d] < 0", v); return TT_ERR_INVALID_ARGUMENT; }
    int32_t p = parent[v];
    if (p < -1 || p >= n || p == v) { set_error("tt_pack: parent[%d] = %d is not a valid parent", v, p); return TT_ERR_NOT_A_FOREST; }
    if (p >= 0) child_cnt[p + 1]++;
    total += len[v];
  }
  if (total == 0) { set_error("tt_pack: the forest has no tokens"); return TT_ERR_EMPTY; }
  if (total > (int64_t)INT32_MAX - 2 * kBlock) { set_error("tt_pack: %lld tokens overflow int32", (long long)total); return TT_ERR_TOO_LARGE; }
  // children CSR, ascending ids (counting sort over ascending v)
  for (int32_t v = 0; v < n; ++v) child_cnt[v + 1] += child_cnt[v];
  std::vector<int32_t> kids(std::max<int64_t>(child_cnt[n], 1));
  {
    std::vector<int32_t> fill(child_cnt.begin(), child_cnt.end() - 1);
    for (int32_t v = 0; v < n; ++v)
      if (parent[v] >= 0) kids[fill[parent[v]]++] = v;
  }
  H.start.assign(n, 0); H.len.assign(len, len + n); H.sub_end.assign(n, 0);
  H.depth.assign(n, 0); H.leaves.assign(n, 0); H.root_start.assign(n, 0);
  // iterative DFS pre-order
  std::vector<int32_t> pre;
  pre.reserve(n);
  std::vector<int32_t> st;
  std::vector<int32_t> next_child(n, 0);
  int64_t cursor = 0;
  for (int32_t r = 0; r < n; ++r) {
    if (parent[r] != -1) continue;
    H.n_roots++;
    st.push_back(r);
    H.depth[r] = 0;
    H.start[r] = (int32_t)cursor;
    H.root_start[r] = (int32_t)cursor;
    cursor += len[r];
    pre.push_back(r);
    while (!st.empty()) {
      int32_t u = st.back();
      int32_t c0 = child_cnt[u], c1 = child_cnt[u + 1];
      if (next_child[u] < c1 - c0) {
        int32_t c = kids[c0 + next_child[u]++];
        H.depth[c] = H.depth[u] + len[u];
        H.start[c] = (int32_t)cursor;
        H.root_start[c] = H.root_start[r];
        cursor += len[c];
        pre.push_back(c);
        st.push_back(c);
        if ((int64_t)pre.size() > n) { set_error("tt_pack: cycle detected"); return TT_ERR_NOT_A_FOREST; }
      } else {
        H.sub_end[u] = (int32_t)cursor;
        st.pop_back();
      }
    }
  }
  if ((int32_t)pre.size() != n) { set_error("tt_pack: %d nodes unreachable from a root (cycle)", n - (int32_t)pre.size()); return TT_ERR_NOT_A_FOREST; }
  H.N = cursor;
  // leaf counts (tree-scale): reverse pre-order accumulates children before parents
  std::vector<int64_t> lv(n, 0);
  for (int32_t t = n - 1; t >= 0; --t) {
    int32_t u = pre[t];
    int64_t s = term ? term[u] : ((child_cnt[u + 1] - child_cnt[u]) == 0 ? 1 : 0);
    for (int32_t c = child_cnt[u]; c < child_cnt[u + 1]; ++c) s += lv[kids[c]];
    lv[u] = s;
  }
  for (int32_t u = 0; u < n; ++u) {
    if (lv[u] > INT32_MAX) { set_error("tt_pack: trajectory count overflows int32"); return TT_ERR_TOO_LARGE; }
    H.leaves[u] = (int32_t)lv[u];
    if (parent[u] == -1) H.n_traj += lv[u];
  }
  // accounting (tokens and allowed pairs, tree vs linearised)
  for (int32_t u = 0; u < n; ++u) {
    int64_t L = len[u], dp = H.depth[u];
    int64_t pr = L * dp + L * (L + 1) / 2;  // sum over the node's tokens of (pos + 1)
    H.lin_tokens += L * lv[u];
    H.pairs += pr;
    H.lin_pairs += pr * lv[u];
  }
  // continuation lists (for the last token of nodes with len > 0), zero-length children recurse
  H.succ_ptr.assign(n + 1, 0);
  H.succ_tok.clear();
  std::vector<int32_t> work;
  for (int32_t u = 0; u < n; ++u) {
    H.succ_ptr[u] = (int32_t)H.succ_tok.size();
    if (len[u] == 0) continue;
    // depth-first over zero-length descendants, children ascending
    work.clear();
    for (int32_t c = child_cnt[u + 1] - 1; c >= child_cnt[u]; --c) work.push_back(kids[c]);
    while (!work.empty()) {
      int32_t c = work.back();
      work.pop_back();
      if (len[c] > 0) {
        H.succ_tok.push_back(H.start[c]);
      } else {
        for (int32_t x = child_cnt[c + 1] - 1; x >= child_cnt[c]; --x) work.push_back(kids[x]);
      }
    }
  }
  H.succ_ptr[n] = (int32_t)H.succ_tok.size();
  H.kids_ptr.assign(child_cnt.begin(), child_cnt.end());
  H.kids.swap(kids);
  H.pre.swap(pre);
  // packed-order list of nodes that own tokens
  H.order.clear(); H.order_start.clear();
  for (int32_t u : H.pre)
    if (len[u] > 0) { H.order.push_back(u); H.order_start.push_back(H.start[u]); }
  return TT_OK;
}

static inline size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

struct PackLayout {
  size_t off_pos, off_w, off_E, off_node, off_kmin, off_kmax, off_fcnt, off_flist;
  size_t off_nodeblk, nodeblk_bytes;
  size_t total;
  int32_t nb;
};

static PackLayout pack_layout(int64_t N, int32_t n, int32_t n_succ, int32_t n_order) {
  PackLayout L{};
  L.nb = (int32_t)ceil_div<int64_t>(N, kBlock);
  size_t o = 0;
  // per-token arrays are padded to whole 128-token blocks (kernels bulk-copy E per block)
  const size_t Np = (size_t)L.nb * kBlock;
  L.off_pos = o; o = al256(o + Np * 4);
  L.off_w = o; o = al256(o + Np * 4);
  L.off_E = o; o = al256(o + Np * 4);
  L.off_node = o; o = al256(o + Np * 4);
  L.off_kmin = o; o = al256(o + (size_t)L.nb * 4);
  L.off_kmax = o; o = al256(o + (size_t)L.nb * 4);
  L.off_fcnt = o; o = al256(o + (size_t)L.nb * 4);
  L.off_flist = o; o = al256(o + (size_t)tri_off(L.nb) * 4);
  // node block: start, len, sub_end, depth, leaves [n] each, succ_ptr [n+1], succ_tok, order, order_start
  L.off_nodeblk = o;
  L.nodeblk_bytes = (size_t)(5 * (size_t)n + (n + 1) + n_succ + 2 * (size_t)n_order + 2 * (size_t)L.nb) * 4;
  o = al256(o + L.nodeblk_bytes);
  L.total = o;
  return L;
}

}  // namespace tt

using namespace tt;

extern "C" {

const char* tt_status_string(tt_status s) {
  switch (s) {
    case TT_OK: return "ok";
    case TT_ERR_INVALID_ARGUMENT: return "invalid argument";
    case TT_ERR_NOT_A_FOREST: return "not a forest";
    case TT_ERR_EMPTY: return "empty";
    case TT_ERR_TOO_LARGE: return "too large";
    case TT_ERR_UNSUPPORTED: return "unsupported";
    case TT_ERR_ALIGNMENT: return "alignment";
    case TT_ERR_WORKSPACE: return "workspace too small";
    case TT_ERR_CUDA: return "cuda error";
  }
  return "unknown";
}

const char* tt_last_error(void) { return g_err.c_str(); }
int32_t tt_version(void) { return 100; }
int32_t tt_build_flags(void) { return tt::kDevBuild ? TT_BUILD_DEV : 0; }
int64_t tt_launch_count(void) { return g_launches; }
void tt_launch_count_reset(void) { g_launches = 0; }

tt_status tt_pack_plan(const int32_t* parent, const int32_t* len, const int32_t* term, int32_t n_nodes,
                       tt_pack_info* info) {
  clear_error();
  if (!info) { set_error("tt_pack_plan: info is null"); return TT_ERR_INVALID_ARGUMENT; }
  HostPack H;
  tt_status s = host_pack(parent, len, term, n_nodes, H);
  if (s) return s;
  PackLayout L = pack_layout(H.N, H.n, (int32_t)H.succ_tok.size(), (int32_t)H.order.size());
  if (H.n_traj > INT32_MAX) { set_error("tt_pack_plan: too many trajectories"); return TT_ERR_TOO_LARGE; }
  info->n_nodes = H.n;
  info->n_roots = H.n_roots;
  info->n_traj = (int32_t)H.n_traj;
  info->n_blk = L.nb;
  info->n_succ = (int32_t)H.succ_tok.size();
  info->reserved = 0;
  info->n_tokens = H.N;
  info->n_linear_tokens = H.lin_tokens;
  info->n_pairs = H.pairs;
  info->n_linear_pairs = H.lin_pairs;
  info->ws_bytes = L.total;
  return TT_OK;
}

// Host -> device copy of a host-built image through a per-thread ring of pinned staging buffers
// (a copy from pageable memory would synchronise the stream).  A slot is rewritten only after the
// event recorded behind its previous copy has completed.  Staging a host image is not capturable
// (a graph would replay whatever the slot holds then), so a capturing stream is refused.
static tt_status stage_h2d(void* dst, const void* src, size_t bytes, cudaStream_t st, const char* who) {
  struct Slot { void* buf = nullptr; size_t cap = 0; cudaEvent_t ev = nullptr; bool used = false; };
  struct Ring {
    Slot slot[4];
    int next = 0;
    ~Ring() {
      // thread exit: release what this thread staged through (errors ignored at process teardown)
      for (Slot& s : slot) {
        if (s.ev) { cudaEventSynchronize(s.ev); cudaEventDestroy(s.ev); }
        if (s.buf) cudaFreeHost(s.buf);
      }
      cudaGetLastError();
    }
  };
  thread_local Ring ring;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    set_error("%s: stages host data and cannot be captured into a CUDA graph (call it outside the capture)", who);
    return TT_ERR_INVALID_ARGUMENT;
  }
  Slot& s = ring.slot[ring.next];
  ring.next = (ring.next + 1) % 4;
  if (s.used && cudaEventSynchronize(s.ev) != cudaSuccess) {
    set_error("%s: staging event: %s", who, cudaGetErrorString(cudaGetLastError()));
    return TT_ERR_CUDA;
  }
  if (s.cap < bytes) {
    if (s.buf) cudaFreeHost(s.buf);
    s.buf = nullptr;
    s.cap = 0;
    const size_t cap = std::max<size_t>(bytes, 1 << 16);
    if (cudaHostAlloc(&s.buf, cap, cudaHostAllocDefault) != cudaSuccess) {
      set_error("%s: pinned staging buffer (%zu bytes): %s", who, cap, cudaGetErrorString(cudaGetLastError()));
      return TT_ERR_CUDA;
    }
    s.cap = cap;
  }
  if (!s.ev && cudaEventCreateWithFlags(&s.ev, cudaEventDisableTiming) != cudaSuccess) {
    set_error("%s: staging event: %s", who, cudaGetErrorString(cudaGetLastError()));
    return TT_ERR_CUDA;
  }
  std::memcpy(s.buf, src, bytes);
  cudaError_t e = cudaMemcpyAsync(dst, s.buf, bytes, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaEventRecord(s.ev, st);
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error("%s: H2D copy failed: %s", who, cudaGetErrorString(e));
    return TT_ERR_CUDA;
  }
  s.used = true;
  return TT_OK;
}

tt_status tt_pack(const int32_t* parent, const int32_t* len, const int32_t* term, int32_t n_nodes, void* d_ws,
                  size_t ws_bytes, tt_packed* out, tt_pack_info* info, tt_stream_t stream) {
  clear_error();
  if (!out || !d_ws) { set_error("tt_pack: out and d_ws must be non-null"); return TT_ERR_INVALID_ARGUMENT; }
  HostPack H;
  tt_status s = host_pack(parent, len, term, n_nodes, H);
  if (s) return s;
  const int32_t n_succ = (int32_t)H.succ_tok.size();
  const int32_t n_order = (int32_t)H.order.size();
  PackLayout L = pack_layout(H.N, H.n, n_succ, n_order);
  if (ws_bytes < L.total) { set_error("tt_pack: workspace %zu < required %zu bytes", ws_bytes, L.total); return TT_ERR_WORKSPACE; }
  if ((reinterpret_cast<uintptr_t>(d_ws) & 255u) != 0) { set_error("tt_pack: d_ws must be 256-byte aligned"); return TT_ERR_ALIGNMENT; }
  char* base = static_cast<char*>(d_ws);
  // node block: one contiguous host image, one async H2D copy
  std::vector<int32_t> img;
  img.reserve(L.nodeblk_bytes / 4);
  const int32_t n = H.n;
  img.insert(img.end(), H.start.begin(), H.start.end());
  img.insert(img.end(), H.len.begin(), H.len.end());
  img.insert(img.end(), H.sub_end.begin(), H.sub_end.end());
  img.insert(img.end(), H.depth.begin(), H.depth.end());
  img.insert(img.end(), H.leaves.begin(), H.leaves.end());
  img.insert(img.end(), H.succ_ptr.begin(), H.succ_ptr.end());
  img.insert(img.end(), H.succ_tok.begin(), H.succ_tok.end());
  img.insert(img.end(), H.order.begin(), H.order.end());
  img.insert(img.end(), H.order_start.begin(), H.order_start.end());
  // per q-block: the first k-block of the tree holding the block's first token (no key of an
  // earlier tree is ever visible, so the tile classification of a forest starts there)
  // and per block the packed-order index of the node holding its first token (pack_fill_kernel's start)
  std::vector<int32_t> blk_first_h(L.nb);
  for (int32_t qb = 0; qb < L.nb; ++qb) {
    const int32_t i0 = qb * kBlock;
    const int32_t k = (int32_t)(std::upper_bound(H.order_start.begin(), H.order_start.end(), i0) - H.order_start.begin()) - 1;
    img.push_back(H.root_start[H.order[std::max(k, 0)]] / kBlock);
    blk_first_h[qb] = std::max(k, 0);
  }
  img.insert(img.end(), blk_first_h.begin(), blk_first_h.end());
  int32_t* nb = reinterpret_cast<int32_t*>(base + L.off_nodeblk);
  cudaStream_t st = as_cuda(stream);
  if ((s = stage_h2d(nb, img.data(), img.size() * 4, st, "tt_pack"))) return s;
  tt_packed P{};
  P.pos = reinterpret_cast<int32_t*>(base + L.off_pos);
  P.w = reinterpret_cast<int32_t*>(base + L.off_w);
  P.E = reinterpret_cast<int32_t*>(base + L.off_E);
  P.node = reinterpret_cast<int32_t*>(base + L.off_node);
  P.node_start = nb;
  P.node_len = nb + n;
  P.node_sub_end = nb + 2 * n;
  P.node_depth = nb + 3 * n;
  P.node_leaves = nb + 4 * n;
  P.succ_ptr = nb + 5 * n;
  P.succ_tok = nb + 6 * n + 1;
  const int32_t* order = nb + 6 * n + 1 + n_succ;
  const int32_t* order_start = order + n_order;
  const int32_t* kb_lo = order_start + n_order;
  const int32_t* blk_first = kb_lo + L.nb;
  P.kblk_minE = reinterpret_cast<int32_t*>(base + L.off_kmin);
  P.kblk_maxE = reinterpret_cast<int32_t*>(base + L.off_kmax);
  P.fwd_cnt = reinterpret_cast<int32_t*>(base + L.off_fcnt);
  P.fwd_list = reinterpret_cast<int32_t*>(base + L.off_flist);
  P.n_tokens = H.N;
  P.n_nodes = n;
  P.n_blk = L.nb;
  P.n_succ = n_succ;
  P.max_succ = 0;
  for (int32_t u = 0; u < n; ++u) P.max_succ = std::max(P.max_succ, H.succ_ptr[u + 1] - H.succ_ptr[u]);
  {
    // per 128-key block the largest subtree end of the nodes it holds (= kblk_maxE, which the device
    // also writes), then the backward's per-block query-tile counts (CTA-order statistics)
    std::vector<int32_t> bmax(L.nb, 0);
    for (int32_t u : H.order) {
      const int32_t b0 = H.start[u] / kBlock, b1 = (H.start[u] + H.len[u] - 1) / kBlock;
      for (int32_t b = b0; b <= b1; ++b) bmax[b] = std::max(bmax[b], H.sub_end[u]);
    }
    P.sched_sum_nq = 0;
    P.sched_max_nq = 0;
    for (int32_t b = 0; b < L.nb; ++b) {
      const int32_t nq = (bmax[b] + 63) / 64 - 2 * b;
      P.sched_sum_nq += nq;
      P.sched_max_nq = std::max(P.sched_max_nq, nq);
    }
    P.wr_negative = 0;
  }
  s = launch_pack_fill(P, order, order_start, n_order, kb_lo, blk_first, const_cast<int32_t*>(P.pos), const_cast<int32_t*>(P.w),
                       const_cast<int32_t*>(P.E), const_cast<int32_t*>(P.node), const_cast<int32_t*>(P.kblk_minE),
                       const_cast<int32_t*>(P.kblk_maxE), const_cast<int32_t*>(P.fwd_cnt),
                       const_cast<int32_t*>(P.fwd_list), st);
  if (s) return s;
  *out = P;
  if (info) {
    info->n_nodes = n; info->n_roots = H.n_roots; info->n_traj = (int32_t)H.n_traj; info->n_blk = L.nb;
    info->n_succ = n_succ; info->reserved = 0; info->n_tokens = H.N; info->n_linear_tokens = H.lin_tokens;
    info->n_pairs = H.pairs; info->n_linear_pairs = H.lin_pairs; info->ws_bytes = L.total;
  }
  return TT_OK;
}

tt_status tt_pack_weights(const int32_t* parent, const int32_t* len, const int32_t* term, int32_t n_nodes,
                          const float* traj_weight, tt_packed* pk, float* wr, tt_stream_t stream) {
  clear_error();
  if (!pk || !wr || !traj_weight) { set_error("tt_pack_weights: pk, traj_weight and wr must be non-null"); return TT_ERR_INVALID_ARGUMENT; }
  if ((reinterpret_cast<uintptr_t>(wr) & 15u) != 0) { set_error("tt_pack_weights: wr must be 16-byte aligned"); return TT_ERR_ALIGNMENT; }
  HostPack H;
  tt_status s = host_pack(parent, len, term, n_nodes, H);
  if (s) return s;
  if (H.n != pk->n_nodes || H.N != pk->n_tokens) {
    set_error("tt_pack_weights: forest (n=%d, N=%lld) is not the one pk was packed from (n=%d, N=%lld)", H.n,
              (long long)H.N, pk->n_nodes, (long long)pk->n_tokens);
    return TT_ERR_INVALID_ARGUMENT;
  }
  const int32_t n = H.n;
  // alpha summed per end node in canonical trajectory order (pre-order, term copies consecutive),
  // then subtree sums in reverse pre-order, all in fp64
  std::vector<double> W(n, 0.0);
  int64_t k = 0;
  for (int32_t u : H.pre) {
    const int64_t t = term ? term[u] : ((H.kids_ptr[u + 1] == H.kids_ptr[u]) ? 1 : 0);
    for (int64_t c = 0; c < t; ++c, ++k) {
      const float a = traj_weight[k];
      if (!std::isfinite(a)) { set_error("tt_pack_weights: traj_weight[%lld] is not finite", (long long)k); return TT_ERR_INVALID_ARGUMENT; }
      W[u] += (double)a;
    }
  }
  for (int32_t t = n - 1; t >= 0; --t) {
    const int32_t u = H.pre[t];
    for (int32_t c = H.kids_ptr[u]; c < H.kids_ptr[u + 1]; ++c) W[u] += W[H.kids[c]];
  }
  const int64_t Np = (int64_t)pk->n_blk * kBlock;
  std::vector<float> img((size_t)Np, 0.f);
  int32_t negative = 0;
  for (int32_t u = 0; u < n; ++u) {
    const float wu = (float)W[u];
    if (H.len[u] > 0 && wu < 0.f) negative = 1;
    for (int32_t i = H.start[u]; i < H.start[u] + H.len[u]; ++i) img[i] = wu;
  }
  if (tt_status s2 = stage_h2d(wr, img.data(), img.size() * 4, as_cuda(stream), "tt_pack_weights")) return s2;
  pk->wr = wr;
  pk->wr_negative = negative;
  return TT_OK;
}

static tt_status check_attn_args(const char* who, const tt_packed* pk, tt_dtype dt, int hq, int hkv, int d) {
  if (!pk) { set_error("%s: pk is null", who); return TT_ERR_INVALID_ARGUMENT; }
  if (pk->n_tokens <= 0) { set_error("%s: empty pack", who); return TT_ERR_EMPTY; }
  if (hq <= 0 || hkv <= 0 || hq % hkv) { set_error("%s: need hq %% hkv == 0 (hq=%d hkv=%d)", who, hq, hkv); return TT_ERR_UNSUPPORTED; }
  if (dt != TT_BF16 && dt != TT_FP32) { set_error("%s: bad dtype %d", who, (int)dt); return TT_ERR_INVALID_ARGUMENT; }
  bool ok = (d == 128 && dt == TT_BF16) || (d == 64) || (d == 128 && dt == TT_FP32);
  if (!ok) { set_error("%s: unsupported (d=%d, dtype=%d)", who, d, (int)dt); return TT_ERR_UNSUPPORTED; }
  if ((int64_t)pk->n_tokens * hq * d > ((int64_t)1 << 40)) { set_error("%s: tensor too large", who); return TT_ERR_TOO_LARGE; }
  return TT_OK;
}

tt_status tt_attn_fwd(const tt_packed* pk, const void* q, const void* k, const void* v, tt_dtype dt, int32_t hq,
                      int32_t hkv, int32_t d, float softmax_scale, void* o, float* lse, tt_stream_t stream) {
  clear_error();
  tt_status s = check_attn_args("tt_attn_fwd", pk, dt, hq, hkv, d);
  if (s) return s;
  if (!q || !k || !v || !o || !lse) { set_error("tt_attn_fwd: null tensor"); return TT_ERR_INVALID_ARGUMENT; }
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o) || !aligned16(lse)) {
    set_error("tt_attn_fwd: tensors must be 16-byte aligned"); return TT_ERR_ALIGNMENT;
  }
  cudaStream_t st = as_cuda(stream);
  if (dt == TT_BF16 && d == 128) {
    if (!sm100_available()) { set_error("tt_attn_fwd: bf16 d=128 needs an sm_100a device"); return TT_ERR_UNSUPPORTED; }
    return sm100_attn_fwd(*pk, q, k, v, hq, hkv, d, softmax_scale, o, lse, st);
  }
  return simt_attn_fwd(*pk, q, k, v, dt, hq, hkv, d, softmax_scale, o, lse, st);
}

static size_t bwd_ws_bytes(const tt_packed* pk, int hq, int hkv, int d, tt_dtype dt) {
  if (dt == TT_BF16 && d == 128) return sm100_bwd_ws_bytes(pk->n_tokens, hq, hkv, d);
  return al256((size_t)pk->n_tokens * hq * 4) + al256(3 * kSqnormBlocks * sizeof(double));
}

tt_status tt_attn_bwd_workspace(const tt_packed* pk, int32_t hq, int32_t hkv, int32_t d, tt_dtype dt, size_t* bytes) {
  clear_error();
  tt_status s = check_attn_args("tt_attn_bwd_workspace", pk, dt, hq, hkv, d);
  if (s) return s;
  if (!bytes) { set_error("tt_attn_bwd_workspace: bytes is null"); return TT_ERR_INVALID_ARGUMENT; }
  *bytes = bwd_ws_bytes(pk, hq, hkv, d, dt);
  return TT_OK;
}

tt_status tt_attn_bwd_kernel(const tt_packed* pk, int32_t hq, int32_t hkv, int32_t d, tt_dtype dt, int32_t* kernel) {
  clear_error();
  tt_status s = check_attn_args("tt_attn_bwd_kernel", pk, dt, hq, hkv, d);
  if (s) return s;
  if (!kernel) { set_error("tt_attn_bwd_kernel: kernel is null"); return TT_ERR_INVALID_ARGUMENT; }
  *kernel = (dt == TT_BF16 && d == 128) ? (bwd_use_flat(*pk, hq, hkv) ? 1 : 0) : 2;
  return TT_OK;
}

tt_status tt_attn_bwd(const tt_packed* pk, const void* q, const void* k, const void* v, const void* o,
                      const float* lse, const void* dout, int32_t restore, tt_dtype dt, int32_t hq, int32_t hkv,
                      int32_t d, float softmax_scale, void* dq, void* dk, void* dv, double* sqnorm, void* d_ws,
                      size_t ws_bytes, tt_stream_t stream) {
  clear_error();
  tt_status s = check_attn_args("tt_attn_bwd", pk, dt, hq, hkv, d);
  if (s) return s;
  if (!q || !k || !v || !o || !lse || !dout || !dq || !dk || !dv || !d_ws) {
    set_error("tt_attn_bwd: null tensor"); return TT_ERR_INVALID_ARGUMENT;
  }
  const void* ptrs[] = {q, k, v, o, lse, dout, dq, dk, dv, d_ws};
  for (const void* p : ptrs)
    if (!aligned16(p)) { set_error("tt_attn_bwd: tensors must be 16-byte aligned"); return TT_ERR_ALIGNMENT; }
  size_t need = bwd_ws_bytes(pk, hq, hkv, d, dt);
  if (ws_bytes < need) { set_error("tt_attn_bwd: workspace %zu < %zu", ws_bytes, need); return TT_ERR_WORKSPACE; }
  cudaStream_t st = as_cuda(stream);
  if (dt == TT_BF16 && d == 128) {
    if (!sm100_available()) { set_error("tt_attn_bwd: bf16 d=128 needs an sm_100a device"); return TT_ERR_UNSUPPORTED; }
    return sm100_attn_bwd(*pk, q, k, v, o, lse, dout, restore, hq, hkv, d, softmax_scale, d_ws, dq, dk, dv, sqnorm, st);
  }
  float* Dvec = static_cast<float*>(d_ws);
  s = launch_bwd_pre(o, dout, dt, pk->n_tokens, hq, d, Dvec, nullptr, st);
  if (s) return s;
  s = simt_attn_bwd(*pk, q, k, v, lse, Dvec, dout, restore, dt, hq, hkv, d, softmax_scale, dq, dk, dv, st);
  if (s || !sqnorm) return s;
  const void* xs[3] = {dq, dk, dv};
  const int64_t ns[3] = {pk->n_tokens * hq * d, pk->n_tokens * hkv * d, pk->n_tokens * hkv * d};
  double* part = reinterpret_cast<double*>(static_cast<char*>(d_ws) + al256((size_t)pk->n_tokens * hq * 4));
  return launch_sqnorm(xs, ns, 3, dt, sqnorm, part, st);
}

size_t tt_restore_loss_workspace(const tt_packed* pk) {
  if (!pk) return 0;
  return al256((size_t)pk->n_tokens * 4) * 2;
}

tt_status tt_restore_loss(const tt_packed* pk, const void* logits, int64_t ld, int32_t vocab, const int32_t* tok,
                          const uint8_t* node_loss_mask, int32_t boundary_mode, float grad_scale, void* dlogits,
                          float* tok_loss, double* sums, int32_t* d_err, void* d_ws, size_t ws_bytes,
                          tt_stream_t stream) {
  clear_error();
  if (!pk || !logits || !tok || !dlogits || !sums || !d_ws) { set_error("tt_restore_loss: null argument"); return TT_ERR_INVALID_ARGUMENT; }
  if (pk->n_tokens <= 0) { set_error("tt_restore_loss: empty pack"); return TT_ERR_EMPTY; }
  if (vocab <= 0 || ld < vocab) { set_error("tt_restore_loss: need 0 < vocab <= ld"); return TT_ERR_INVALID_ARGUMENT; }
  if (boundary_mode != 0 && boundary_mode != 1) { set_error("tt_restore_loss: boundary_mode must be 0 or 1"); return TT_ERR_INVALID_ARGUMENT; }
  if (!aligned16(logits) || !aligned16(dlogits) || (ld % 8) != 0) {
    set_error("tt_restore_loss: logits/dlogits rows must be 16-byte aligned (ld %% 8 == 0)"); return TT_ERR_ALIGNMENT;
  }
  if (pk->max_succ > 1024) { set_error("tt_restore_loss: a node has %d > 1024 continuations", pk->max_succ); return TT_ERR_UNSUPPORTED; }
  if (ws_bytes < tt_restore_loss_workspace(pk)) { set_error("tt_restore_loss: workspace too small"); return TT_ERR_WORKSPACE; }
  float* ws_loss = static_cast<float*>(d_ws);
  float* ws_omega = reinterpret_cast<float*>(static_cast<char*>(d_ws) + al256((size_t)pk->n_tokens * 4));
  return launch_loss(*pk, static_cast<const __nv_bfloat16*>(logits), ld, vocab, tok, node_loss_mask, boundary_mode,
                     grad_scale, static_cast<__nv_bfloat16*>(dlogits), tok_loss, sums, d_err, ws_loss, ws_omega,
                     as_cuda(stream));
}

size_t tt_grad_sqnorm_workspace(int64_t n) { (void)n; return al256(3 * kSqnormBlocks * sizeof(double)); }

tt_status tt_grad_sqnorm(const void* x, int64_t n, tt_dtype dt, double* out, void* d_ws, size_t ws_bytes,
                         tt_stream_t stream) {
  clear_error();
  if (!x || !out || !d_ws || n < 0) { set_error("tt_grad_sqnorm: bad argument"); return TT_ERR_INVALID_ARGUMENT; }
  if (!aligned16(x)) { set_error("tt_grad_sqnorm: x must be 16-byte aligned"); return TT_ERR_ALIGNMENT; }
  if (dt != TT_BF16 && dt != TT_FP32) { set_error("tt_grad_sqnorm: bad dtype"); return TT_ERR_INVALID_ARGUMENT; }
  if (ws_bytes < tt_grad_sqnorm_workspace(n)) { set_error("tt_grad_sqnorm: workspace too small"); return TT_ERR_WORKSPACE; }
  const void* xs[1] = {x};
  const int64_t ns[1] = {n};
  return launch_sqnorm(xs, ns, 1, dt, out, static_cast<double*>(d_ws), as_cuda(stream));
}

tt_status tt_grad_sqnorm3(const void* x0, int64_t n0, const void* x1, int64_t n1, const void* x2, int64_t n2,
                          tt_dtype dt, double* out, void* d_ws, size_t ws_bytes, tt_stream_t stream) {
  clear_error();
  const void* xs[3] = {x0, x1, x2};
  const int64_t ns[3] = {n0, n1, n2};
  for (int k = 0; k < 3; ++k) {
    if (!xs[k] || ns[k] < 0) { set_error("tt_grad_sqnorm3: bad tensor %d", k); return TT_ERR_INVALID_ARGUMENT; }
    if (!aligned16(xs[k])) { set_error("tt_grad_sqnorm3: tensor %d must be 16-byte aligned", k); return TT_ERR_ALIGNMENT; }
  }
  if (!out || !d_ws) { set_error("tt_grad_sqnorm3: bad argument"); return TT_ERR_INVALID_ARGUMENT; }
  if (dt != TT_BF16 && dt != TT_FP32) { set_error("tt_grad_sqnorm3: bad dtype"); return TT_ERR_INVALID_ARGUMENT; }
  if (ws_bytes < tt_grad_sqnorm_workspace(0)) { set_error("tt_grad_sqnorm3: workspace too small"); return TT_ERR_WORKSPACE; }
  return launch_sqnorm(xs, ns, 3, dt, out, static_cast<double*>(d_ws), as_cuda(stream));
}

tt_status tt_lmhead_loss_workspace(const tt_packed* pk, int32_t hidden, int32_t vocab, int32_t vocab_chunk,
                                   size_t* bytes) {
  clear_error();
  if (!pk || !bytes || hidden <= 0 || vocab <= 0 || vocab_chunk <= 0) { set_error("tt_lmhead_loss_workspace: bad argument"); return TT_ERR_INVALID_ARGUMENT; }
  *bytes = lmhead_ws_bytes(pk->n_tokens, hidden, vocab, vocab_chunk, pk->max_succ);
  return TT_OK;
}

tt_status tt_lmhead_loss(const tt_packed* pk, const void* h, const void* w, int32_t hidden, int32_t vocab,
                         int32_t vocab_chunk, const int32_t* tok, const uint8_t* node_loss_mask, int32_t boundary_mode,
                         float grad_scale, void* dh, void* dw, float* tok_loss, double* sums, int32_t* d_err,
                         void* d_ws, size_t ws_bytes, tt_stream_t stream) {
  clear_error();
  if (!pk || !h || !w || !tok || !dh || !dw || !sums || !d_ws) { set_error("tt_lmhead_loss: null argument"); return TT_ERR_INVALID_ARGUMENT; }
  if (pk->n_tokens <= 0) { set_error("tt_lmhead_loss: empty pack"); return TT_ERR_EMPTY; }
  if (hidden <= 0 || vocab <= 0 || vocab_chunk <= 0) { set_error("tt_lmhead_loss: bad sizes"); return TT_ERR_INVALID_ARGUMENT; }
  if (boundary_mode != 0 && boundary_mode != 1) { set_error("tt_lmhead_loss: boundary_mode must be 0 or 1"); return TT_ERR_INVALID_ARGUMENT; }
  if (hidden % 8 != 0) { set_error("tt_lmhead_loss: hidden must be a multiple of 8"); return TT_ERR_UNSUPPORTED; }
  if (!aligned16(h) || !aligned16(w) || !aligned16(dh) || !aligned16(dw) || !aligned16(d_ws)) {
    set_error("tt_lmhead_loss: tensors must be 16-byte aligned"); return TT_ERR_ALIGNMENT;
  }
  if (pk->n_tokens > INT32_MAX) { set_error("tt_lmhead_loss: too many rows"); return TT_ERR_TOO_LARGE; }
  if (ws_bytes < lmhead_ws_bytes(pk->n_tokens, hidden, vocab, vocab_chunk, pk->max_succ)) { set_error("tt_lmhead_loss: workspace too small"); return TT_ERR_WORKSPACE; }
  return launch_lmhead_loss(*pk, static_cast<const __nv_bfloat16*>(h), static_cast<const __nv_bfloat16*>(w), hidden, vocab,
                            vocab_chunk, tok, node_loss_mask, boundary_mode, grad_scale, static_cast<__nv_bfloat16*>(dh),
                            static_cast<__nv_bfloat16*>(dw), tok_loss, sums, d_err, d_ws, as_cuda(stream));
}

tt_status tt_gemm(int32_t M, int32_t N, int32_t K, const void* a, int64_t lda, int32_t a_mn, const void* b,
                  int64_t ldb, int32_t b_mn, void* d, int64_t ldd, tt_dtype d_dt, int32_t accumulate,
                  tt_stream_t stream) {
  clear_error();
  if (M <= 0 || N <= 0 || K <= 0 || !a || !b || !d) { set_error("tt_gemm: bad argument"); return TT_ERR_INVALID_ARGUMENT; }
  if (d_dt != TT_BF16 && d_dt != TT_FP32) { set_error("tt_gemm: bad output dtype"); return TT_ERR_INVALID_ARGUMENT; }
  if (d_dt == TT_BF16 && accumulate) { set_error("tt_gemm: accumulate needs an fp32 output"); return TT_ERR_UNSUPPORTED; }
  if (lda < (a_mn ? M : K) || ldb < (b_mn ? N : K) || ldd < N) { set_error("tt_gemm: leading dimension too small"); return TT_ERR_INVALID_ARGUMENT; }
  if (!aligned16(a) || !aligned16(b) || !aligned16(d) || (lda % 8) || (ldb % 8)) {
    set_error("tt_gemm: operands must be 16-byte aligned with row strides a multiple of 8 elements"); return TT_ERR_ALIGNMENT;
  }
  gemm::GemmEpilogue ep{};
  ep.out = d;
  ep.ldo = ldd;
  ep.beta = accumulate ? 1 : 0;
  return gemm::gemm_run(d_dt == TT_BF16 ? gemm::kEpiStoreBF16 : gemm::kEpiAccF32, M, N, K, a, lda, a_mn ? 1 : 0, b, ldb,
                        b_mn ? 1 : 0, ep, as_cuda(stream));
}

tt_status tt_rope(const tt_packed* pk, void* x, tt_dtype dt, int32_t n_heads, int32_t d, double base,
                  int32_t inverse, tt_stream_t stream) {
  clear_error();
  if (!pk || !x || !pk->pos || n_heads <= 0 || !(base > 0.0)) { set_error("tt_rope: bad argument"); return TT_ERR_INVALID_ARGUMENT; }
  if (dt != TT_BF16 && dt != TT_FP32) { set_error("tt_rope: bad dtype"); return TT_ERR_INVALID_ARGUMENT; }
  if (d != 64 && d != 128) { set_error("tt_rope: head_dim %d unsupported (64, 128)", d); return TT_ERR_UNSUPPORTED; }
  if (!aligned16(x)) { set_error("tt_rope: x must be 16-byte aligned"); return TT_ERR_ALIGNMENT; }
  return launch_rope(*pk, x, dt, n_heads, d, base, inverse, as_cuda(stream));
}

tt_status tt_restore_grad(const tt_packed* pk, void* g, tt_dtype dt, int64_t row_elems, tt_stream_t stream) {
  clear_error();
  if (!pk || !g || !pk->w || row_elems <= 0) { set_error("tt_restore_grad: bad argument"); return TT_ERR_INVALID_ARGUMENT; }
  if (dt != TT_BF16 && dt != TT_FP32) { set_error("tt_restore_grad: bad dtype"); return TT_ERR_INVALID_ARGUMENT; }
  if (row_elems % (dt == TT_BF16 ? 8 : 4)) { set_error("tt_restore_grad: row_elems must be a multiple of 16 bytes"); return TT_ERR_ALIGNMENT; }
  if (!aligned16(g)) { set_error("tt_restore_grad: g must be 16-byte aligned"); return TT_ERR_ALIGNMENT; }
  return launch_restore_grad(*pk, g, dt, row_elems, as_cuda(stream));
}

}  // extern "C"
