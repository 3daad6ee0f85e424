// plan.cu — capacity-constrained Tree Packing (§2.2).
//
// When a tree does not fit the per-GPU token budget C, Tree Packing splits its trajectories into
// traversals (training steps); each traversal is packed as the sub-forest induced by its
// trajectories, so its cost is the number of distinct tokens on their root paths and must be <= C
// (the feasibility constraint of Eq. 3, generalised to multi-path traversals).  The exact
// multi-path DP (Eqs. 6-11) is exponential ("tractable only for small to medium trees",
// P:299); the paper scales with a heuristic:
//   "prioritizes allocating the deepest leaves first ..., groups leaves of similar depths within
//    each subtree ..., and traverses the tree in depth-first order, initiating a new traversal
//    whenever the accumulated length exceeds capacity C."
// Reading (R19): trajectories are visited in DFS order where the children of every node
// are taken in descending order of their deepest trajectory end (ties: ascending id), so deep
// subtrees come first and siblings of similar depth are adjacent; each trajectory joins the current
// traversal if the traversal's induced token count plus the tokens of its path not yet covered stays
// <= C, else a new traversal starts.  Host-only, O(sum of path lengths in nodes).
#include <algorithm>
#include <vector>

#include "tt_internal.cuh"

namespace tt {
namespace {

struct PlanForest {
  int32_t n = 0;
  std::vector<int32_t> kids_ptr, kids;    // children CSR (ascending id)
  std::vector<int32_t> roots;
  std::vector<int64_t> term;
  std::vector<int64_t> depth_end;          // tokens on the root path through the node, inclusive
};

tt_status build(const int32_t* parent, const int32_t* len, const int32_t* term, int32_t n, PlanForest& F) {
  if (!parent || !len || n <= 0) { set_error("tt_plan: parent/len must be non-null, n > 0"); return TT_ERR_INVALID_ARGUMENT; }
  F.n = n;
  F.kids_ptr.assign(n + 1, 0);
  for (int32_t v = 0; v < n; ++v) {
    const int32_t p = parent[v];
    if (len[v] < 0 || (term && term[v] < 0)) { set_error("tt_plan: negative len/term at %d", v); return TT_ERR_INVALID_ARGUMENT; }
    if (p < -1 || p >= n || p == v) { set_error("tt_plan: parent[%d] = %d invalid", v, p); return TT_ERR_NOT_A_FOREST; }
    if (p >= 0) F.kids_ptr[p + 1]++;
  }
  for (int32_t v = 0; v < n; ++v) F.kids_ptr[v + 1] += F.kids_ptr[v];
  F.kids.assign(std::max<int32_t>(F.kids_ptr[n], 1), 0);
  std::vector<int32_t> fill(F.kids_ptr.begin(), F.kids_ptr.end() - 1);
  for (int32_t v = 0; v < n; ++v) {
    if (parent[v] >= 0) F.kids[fill[parent[v]]++] = v;
    else F.roots.push_back(v);
  }
  F.term.assign(n, 0);
  for (int32_t v = 0; v < n; ++v)
    F.term[v] = term ? term[v] : ((F.kids_ptr[v + 1] == F.kids_ptr[v]) ? 1 : 0);
  // depth (inclusive) by iterative DFS; detects cycles as unreachable nodes
  F.depth_end.assign(n, -1);
  std::vector<int32_t> st;
  int32_t seen = 0;
  for (int32_t r : F.roots) {
    F.depth_end[r] = len[r];
    st.push_back(r);
    while (!st.empty()) {
      const int32_t u = st.back();
      st.pop_back();
      ++seen;
      for (int32_t k = F.kids_ptr[u]; k < F.kids_ptr[u + 1]; ++k) {
        const int32_t c = F.kids[k];
        F.depth_end[c] = F.depth_end[u] + len[c];
        st.push_back(c);
      }
    }
  }
  if (seen != n) { set_error("tt_plan: %d nodes unreachable from a root (cycle)", n - seen); return TT_ERR_NOT_A_FOREST; }
  return TT_OK;
}

// trajectories in canonical order: DFS pre-order (roots / children ascending id) of end nodes,
// term(u) consecutive copies — the order the oracle and tt_pack's tree-scale use
void canonical_trajectories(const PlanForest& F, std::vector<int32_t>& traj_node) {
  traj_node.clear();
  std::vector<int32_t> st;
  for (auto it = F.roots.rbegin(); it != F.roots.rend(); ++it) st.push_back(*it);
  while (!st.empty()) {
    const int32_t u = st.back();
    st.pop_back();
    for (int64_t k = 0; k < F.term[u]; ++k) traj_node.push_back(u);
    for (int32_t k = F.kids_ptr[u + 1] - 1; k >= F.kids_ptr[u]; --k) st.push_back(F.kids[k]);
  }
}

}  // namespace
}  // namespace tt

using namespace tt;

extern "C" {

tt_status tt_plan_traversals(const int32_t* parent, const int32_t* len, const int32_t* term, int32_t n_nodes,
                             int64_t capacity, int32_t* traversal_of_traj, tt_plan_info* info) {
  clear_error();
  if (!info) { set_error("tt_plan_traversals: info is null"); return TT_ERR_INVALID_ARGUMENT; }
  if (capacity <= 0) { set_error("tt_plan_traversals: capacity must be > 0"); return TT_ERR_INVALID_ARGUMENT; }
  PlanForest F;
  tt_status s = build(parent, len, term, n_nodes, F);
  if (s) return s;
  const int32_t n = F.n;
  // deepest trajectory end below each node (post-order via reverse DFS order)
  std::vector<int32_t> order;
  {
    std::vector<int32_t> st(F.roots.begin(), F.roots.end());
    while (!st.empty()) {
      const int32_t u = st.back();
      st.pop_back();
      order.push_back(u);
      for (int32_t k = F.kids_ptr[u]; k < F.kids_ptr[u + 1]; ++k) st.push_back(F.kids[k]);
    }
  }
  std::vector<int64_t> deepest(n, -1);
  for (auto it = order.rbegin(); it != order.rend(); ++it) {
    const int32_t u = *it;
    int64_t d = F.term[u] > 0 ? F.depth_end[u] : -1;
    for (int32_t k = F.kids_ptr[u]; k < F.kids_ptr[u + 1]; ++k) d = std::max(d, deepest[F.kids[k]]);
    deepest[u] = d;
  }
  // canonical trajectory indices (for the output array)
  std::vector<int32_t> canon;
  canonical_trajectories(F, canon);
  const int64_t n_traj = (int64_t)canon.size();
  if (n_traj > INT32_MAX) { set_error("tt_plan_traversals: too many trajectories"); return TT_ERR_TOO_LARGE; }
  std::vector<int64_t> first_idx(n, -1);  // canonical index of the first trajectory ending at u
  for (int64_t k = n_traj - 1; k >= 0; --k) first_idx[canon[k]] = k;
  int64_t lin = 0;
  for (int32_t u : canon) lin += F.depth_end[u];
  for (int32_t u : canon)
    if (F.depth_end[u] > capacity) {
      set_error("tt_plan_traversals: a trajectory of %lld tokens exceeds capacity %lld", (long long)F.depth_end[u],
                (long long)capacity);
      return TT_ERR_TOO_LARGE;
    }
  // heuristic visiting order: DFS, children by descending deepest end (ties ascending id)
  std::vector<int32_t> visit;  // trajectory end nodes in visiting order (term copies consecutive)
  {
    std::vector<int32_t> st, kids;
    std::vector<int32_t> roots = F.roots;
    std::stable_sort(roots.begin(), roots.end(), [&](int32_t a, int32_t b) { return deepest[a] > deepest[b]; });
    for (auto it = roots.rbegin(); it != roots.rend(); ++it) st.push_back(*it);
    while (!st.empty()) {
      const int32_t u = st.back();
      st.pop_back();
      for (int64_t k = 0; k < F.term[u]; ++k) visit.push_back(u);
      kids.assign(F.kids.begin() + F.kids_ptr[u], F.kids.begin() + F.kids_ptr[u + 1]);
      std::stable_sort(kids.begin(), kids.end(), [&](int32_t a, int32_t b) { return deepest[a] > deepest[b]; });
      for (auto it = kids.rbegin(); it != kids.rend(); ++it) st.push_back(*it);
    }
  }
  // greedy fill: a traversal's node set is ancestor-closed, so the new tokens of a trajectory are
  // those of its path nodes up to the first node already in the traversal
  std::vector<int32_t> stamp(n, -1);
  std::vector<int32_t> used(n, 0);  // next unused copy index per end node
  int32_t cur = 0;
  int64_t cur_cost = 0, planned = 0;
  std::vector<int32_t> path;
  for (int32_t u : visit) {
    int64_t add = 0;
    path.clear();
    for (int32_t x = u; x >= 0 && stamp[x] != cur; x = parent[x]) {
      add += len[x];
      path.push_back(x);
    }
    if (cur_cost + add > capacity && cur_cost > 0) {
      planned += cur_cost;
      ++cur;
      cur_cost = 0;
      add = 0;
      path.clear();
      for (int32_t x = u; x >= 0; x = parent[x]) {
        add += len[x];
        path.push_back(x);
      }
    }
    for (int32_t x : path) stamp[x] = cur;
    cur_cost += add;
    const int64_t k = first_idx[u] + used[u]++;
    if (traversal_of_traj) traversal_of_traj[k] = cur;
  }
  planned += cur_cost;
  int64_t tree_tok = 0;
  {
    std::vector<char> on(n, 0);
    for (int32_t u : canon)
      for (int32_t x = u; x >= 0 && !on[x]; x = parent[x]) on[x] = 1;
    for (int32_t v = 0; v < n; ++v)
      if (on[v]) tree_tok += len[v];
  }
  info->n_traj = (int32_t)n_traj;
  info->n_traversals = n_traj ? cur + 1 : 0;
  info->capacity = capacity;
  info->linear_tokens = lin;
  info->tree_tokens = tree_tok;
  info->planned_tokens = planned;
  return TT_OK;
}

tt_status tt_traversal_forest(const int32_t* parent, const int32_t* len, const int32_t* term, int32_t n_nodes,
                              const int32_t* traversal_of_traj, int32_t traversal, int32_t* out_parent,
                              int32_t* out_len, int32_t* out_term, int32_t* out_node, int32_t* n_out) {
  clear_error();
  if (!traversal_of_traj || !out_parent || !out_len || !out_term || !out_node || !n_out) {
    set_error("tt_traversal_forest: null output");
    return TT_ERR_INVALID_ARGUMENT;
  }
  PlanForest F;
  tt_status s = build(parent, len, term, n_nodes, F);
  if (s) return s;
  std::vector<int32_t> canon;
  canonical_trajectories(F, canon);
  std::vector<int32_t> tcount(F.n, 0);
  std::vector<char> on(F.n, 0);
  for (size_t k = 0; k < canon.size(); ++k) {
    if (traversal_of_traj[k] != traversal) continue;
    tcount[canon[k]]++;
    for (int32_t x = canon[k]; x >= 0 && !on[x]; x = parent[x]) on[x] = 1;
  }
  // keep the original relative order of node ids (so DFS orders agree with the full tree)
  std::vector<int32_t> remap(F.n, -1);
  int32_t m = 0;
  for (int32_t v = 0; v < F.n; ++v)
    if (on[v]) { remap[v] = m; out_node[m] = v; ++m; }
  for (int32_t v = 0; v < F.n; ++v) {
    if (!on[v]) continue;
    out_parent[remap[v]] = parent[v] >= 0 ? remap[parent[v]] : -1;
    out_len[remap[v]] = len[v];
    out_term[remap[v]] = tcount[v];
  }
  *n_out = m;
  return TT_OK;
}

}  // extern "C"
