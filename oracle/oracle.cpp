// =====================================================================================
// oracle.cpp — fp64 CPU ORACLE for the Tree Training hot path.  TEST INFRASTRUCTURE ONLY.
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
// load this library.  The product path (paper_2511_00413_b200/, libtt.so) never calls it, and
// the two share no code, headers, tables or helpers.
//
// What it computes is the plain definition the method provably reaches (Eqs. 14-16,
// tree gradients == sum over baseline per-branch gradients):
//   1. pack:  recursive DFS over parent/len (roots ascending, children ascending by id; DESIGN.md
//             reading R3), giving restored position ids, leaf-count weights
//             ("tree-scale", Fig. 4gradient) and subtree ends; plus every
//             trajectory's packed root-to-end index path (x_i = [P;S_i], Eq. 12).
//   2. attention: every trajectory is linearised and ordinary causal softmax attention is run
//             on it row by row (Eq. 1 P:119-126 with an explicit softmax scale, reading R1);
//             tree outputs are scattered back with a BITWISE equality assertion (P:140,
//             "the outputs O1 and O1' are identical").
//   3. backward: per branch, ordinary attention backward (Eq. 2 P:130-135 for dV, standard
//             softmax-attention dQ/dK), upstream gradient G per token; branch gradients are
//             summed into the tree arrays in ascending trajectory order (Eq. 16).
//   4. loss:  per branch ordinary next-token cross entropy, summed (reading R7: multi-target at
//             branch points; R8: sum reduction).
//   5. tiles: brute-force tile classification from the parent-walk (ancestor-or-self) mask.
//
// Everything is fp64, -O2, no -ffast-math.  Each exported function returns 0 on success or an
// OE_* error code.  Threads (std::thread) only partition independent heads / rows, so results
// are bitwise deterministic and independent of the thread count.
//
// Parity pins: see tests/test_oracle_*.py and DESIGN.md "Oracle pins".
// =====================================================================================
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <thread>
#include <vector>

namespace {

enum {
  OE_OK = 0,
  OE_INVALID = 1,     // negative length / term, null pointer, n <= 0
  OE_NOT_FOREST = 2,  // parent out of range, self-parent, cycle
  OE_EMPTY = 3,       // zero tokens in the whole forest
  OE_TOO_LARGE = 4,   // token count overflows int32
  OE_INVARIANT = 5,   // the forward branch-invariance assertion failed (must never happen)
};

struct Forest {
  int n = 0;
  const int32_t* parent = nullptr;
  const int32_t* len = nullptr;
  std::vector<int64_t> term;                // trajectories ending at each node
  std::vector<std::vector<int32_t>> kids;   // children, ascending id
  std::vector<int32_t> roots;               // ascending id
};

// Build + validate.  A cycle is detected as "some node is not reachable from a root".
int build_forest(const int32_t* parent, const int32_t* len, const int32_t* term, int32_t n, Forest& F) {
  if (!parent || !len || n <= 0) return OE_INVALID;
  F.n = n; F.parent = parent; F.len = len;
  F.kids.assign(n, {});
  F.roots.clear();
  for (int v = 0; v < n; ++v) {
    if (len[v] < 0) return OE_INVALID;
    if (term && term[v] < 0) return OE_INVALID;
    int p = parent[v];
    if (p < -1 || p >= n || p == v) return OE_NOT_FOREST;
    if (p == -1) F.roots.push_back(v); else F.kids[p].push_back(v);
  }
  // ids are visited in ascending order above, so kids / roots are already ascending.
  std::vector<char> seen(n, 0);
  int reached = 0;
  std::vector<int32_t> st;
  for (int r : F.roots) {
    st.push_back(r);
    while (!st.empty()) {
      int u = st.back(); st.pop_back();
      if (seen[u]) return OE_NOT_FOREST;
      seen[u] = 1; ++reached;
      for (int c : F.kids[u]) st.push_back(c);
    }
  }
  if (reached != n) return OE_NOT_FOREST;
  F.term.assign(n, 0);
  for (int v = 0; v < n; ++v)
    F.term[v] = term ? term[v] : (F.kids[v].empty() ? 1 : 0);
  return OE_OK;
}

struct PackOut {
  int64_t N = 0;
  std::vector<int32_t> pos, w, E, node;                 // per token
  std::vector<int32_t> start, sub_end, depth, leaves;   // per node
  std::vector<int64_t> path_ptr;                        // trajectories CSR
  std::vector<int32_t> path_idx;
};

// Recursive DFS pre-order (the literal definition of the DFS flattening, Eq. 13).
struct Packer {
  const Forest& F;
  PackOut& P;
  std::vector<int32_t> path;  // packed indices of the current root path
  explicit Packer(const Forest& f, PackOut& p) : F(f), P(p) {}

  int64_t subtree_term(int u) {
    int64_t s = F.term[u];
    for (int c : F.kids[u]) s += subtree_term(c);
    return s;
  }

  void visit(int u, int32_t depth_tokens) {
    P.start[u] = (int32_t)P.N;
    P.depth[u] = depth_tokens;
    P.leaves[u] = (int32_t)subtree_term(u);
    for (int32_t t = 0; t < F.len[u]; ++t) {
      P.pos.push_back(depth_tokens + t);
      P.w.push_back(P.leaves[u]);
      P.E.push_back(-1);  // filled after the subtree is emitted
      P.node.push_back(u);
      path.push_back((int32_t)P.N);
      ++P.N;
    }
    // trajectories ending at u: their path is the current root path
    for (int64_t k = 0; k < F.term[u]; ++k) {
      for (int32_t idx : path) P.path_idx.push_back(idx);
      P.path_ptr.push_back((int64_t)P.path_idx.size());
    }
    for (int c : F.kids[u]) visit(c, depth_tokens + F.len[u]);
    P.sub_end[u] = (int32_t)P.N;
    for (int32_t i = P.start[u]; i < P.start[u] + F.len[u]; ++i) P.E[i] = P.sub_end[u];
    path.resize(path.size() - F.len[u]);
  }

  void run() {
    P.start.assign(F.n, 0); P.sub_end.assign(F.n, 0); P.depth.assign(F.n, 0); P.leaves.assign(F.n, 0);
    P.path_ptr.assign(1, 0);
    for (int r : F.roots) visit(r, 0);
  }
};

int do_pack(const int32_t* parent, const int32_t* len, const int32_t* term, int32_t n, PackOut& P) {
  Forest F;
  int rc = build_forest(parent, len, term, n, F);
  if (rc) return rc;
  int64_t total = 0;
  for (int v = 0; v < n; ++v) total += len[v];
  if (total == 0) return OE_EMPTY;
  if (total > INT32_MAX) return OE_TOO_LARGE;
  Packer pk(F, P);
  pk.run();
  return OE_OK;
}

void run_threads(int n_tasks, int nthreads, const std::function<void(int)>& fn) {
  if (nthreads <= 1 || n_tasks <= 1) {
    for (int t = 0; t < n_tasks; ++t) fn(t);
    return;
  }
  nthreads = std::min(nthreads, n_tasks);
  std::vector<std::thread> th;
  for (int i = 0; i < nthreads; ++i)
    th.emplace_back([&, i]() { for (int t = i; t < n_tasks; t += nthreads) fn(t); });
  for (auto& x : th) x.join();
}

// One row of ordinary causal attention on a linearised branch (Eq. 1), computed exactly as the
// textbook definition with max subtraction:  s_j = scale * q.k_j (j <= p), m = max s,
// l = sum exp(s_j - m), o = sum exp(s_j - m)/l * v_j, lse = m + ln l.
void attn_row(const double* q, const double* const* krows, const double* const* vrows, int n_keys,
              int d, double scale, std::vector<double>& s, double* o, double* lse) {
  s.resize(n_keys);
  double m = -INFINITY;
  for (int j = 0; j < n_keys; ++j) {
    double acc = 0.0;
    for (int c = 0; c < d; ++c) acc += q[c] * krows[j][c];
    s[j] = scale * acc;
    m = std::max(m, s[j]);
  }
  double l = 0.0;
  for (int j = 0; j < n_keys; ++j) l += std::exp(s[j] - m);
  for (int c = 0; c < d; ++c) o[c] = 0.0;
  for (int j = 0; j < n_keys; ++j) {
    double p = std::exp(s[j] - m) / l;
    for (int c = 0; c < d; ++c) o[c] += p * vrows[j][c];
  }
  *lse = m + std::log(l);
}

}  // namespace

extern "C" {

// ---------------------------------------------------------------------------------------------
// Pack.  Call once with null outputs to get sizes, then again with buffers of those sizes.
// ---------------------------------------------------------------------------------------------
int oracle_pack_sizes(const int32_t* parent, const int32_t* len, const int32_t* term, int32_t n,
                      int64_t* n_tokens, int64_t* n_traj, int64_t* n_path_tokens) {
  PackOut P;
  int rc = do_pack(parent, len, term, n, P);
  if (rc) return rc;
  *n_tokens = P.N;
  *n_traj = (int64_t)P.path_ptr.size() - 1;
  *n_path_tokens = (int64_t)P.path_idx.size();
  return OE_OK;
}

int oracle_pack(const int32_t* parent, const int32_t* len, const int32_t* term, int32_t n,
                int32_t* pos, int32_t* w, int32_t* E, int32_t* node,
                int32_t* node_start, int32_t* node_sub_end, int32_t* node_depth, int32_t* node_leaves,
                int64_t* path_ptr, int32_t* path_idx) {
  PackOut P;
  int rc = do_pack(parent, len, term, n, P);
  if (rc) return rc;
  std::memcpy(pos, P.pos.data(), P.N * 4);
  std::memcpy(w, P.w.data(), P.N * 4);
  std::memcpy(E, P.E.data(), P.N * 4);
  std::memcpy(node, P.node.data(), P.N * 4);
  std::memcpy(node_start, P.start.data(), n * 4);
  std::memcpy(node_sub_end, P.sub_end.data(), n * 4);
  std::memcpy(node_depth, P.depth.data(), n * 4);
  std::memcpy(node_leaves, P.leaves.data(), n * 4);
  std::memcpy(path_ptr, P.path_ptr.data(), P.path_ptr.size() * 8);
  std::memcpy(path_idx, P.path_idx.data(), P.path_idx.size() * 4);
  return OE_OK;
}

// ---------------------------------------------------------------------------------------------
// Dense shared-prefix mask by the definition (SPEC): token i may attend j iff node(j) is an
// ancestor-or-self of node(i) (parent walk) and pos_j <= pos_i.  Written row-major [N, N].
// Only for small N (tests).
// ---------------------------------------------------------------------------------------------
int oracle_dense_mask(const int32_t* parent, int32_t n, int64_t N, const int32_t* node,
                      const int32_t* pos, uint8_t* mask) {
  for (int64_t i = 0; i < N; ++i) {
    for (int64_t j = 0; j < N; ++j) {
      int a = node[j];
      bool anc = false;
      for (int u = node[i]; u >= 0; u = parent[u]) {
        if (u < 0 || u >= n) return OE_NOT_FOREST;
        if (u == a) { anc = true; break; }
      }
      mask[i * N + j] = (anc && pos[j] <= pos[i]) ? 1 : 0;
    }
  }
  return OE_OK;
}

// ---------------------------------------------------------------------------------------------
// Brute-force tile classification (B x B tiles over the packed sequence) from the parent-walk
// ancestor relation.  cls[qb * nb + kb] = 0 empty, 1 partial, 2 full (full = every (i, j) of the
// tile clipped to [0, N) is allowed).  Also per-k-block min/max of E over its keys.
// ---------------------------------------------------------------------------------------------
int oracle_tiles(const int32_t* parent, int32_t n, int64_t N, const int32_t* node, const int32_t* pos,
                 const int32_t* E, int32_t B, uint8_t* cls, int32_t* kblk_minE, int32_t* kblk_maxE) {
  if (B <= 0) return OE_INVALID;
  // ancestor-or-self table over nodes: anc[a * n + u] = a is ancestor-or-self of u
  std::vector<uint8_t> anc((size_t)n * n, 0);
  for (int u = 0; u < n; ++u)
    for (int a = u; a >= 0; a = parent[a]) anc[(size_t)a * n + u] = 1;
  int64_t nb = (N + B - 1) / B;
  for (int64_t qb = 0; qb < nb; ++qb) {
    for (int64_t kb = 0; kb < nb; ++kb) {
      int64_t cnt = 0, tot = 0;
      for (int64_t i = qb * B; i < std::min<int64_t>(N, qb * B + B); ++i)
        for (int64_t j = kb * B; j < std::min<int64_t>(N, kb * B + B); ++j) {
          ++tot;
          bool ok = anc[(size_t)node[j] * n + node[i]] && pos[j] <= pos[i];
          cnt += ok;
        }
      cls[qb * nb + kb] = cnt == 0 ? 0 : (cnt == tot ? 2 : 1);
    }
  }
  for (int64_t kb = 0; kb < nb; ++kb) {
    int32_t mn = INT32_MAX, mx = INT32_MIN;
    for (int64_t j = kb * B; j < std::min<int64_t>(N, kb * B + B); ++j) {
      mn = std::min(mn, E[j]);
      mx = std::max(mx, E[j]);
    }
    kblk_minE[kb] = mn;
    kblk_maxE[kb] = mx;
  }
  return OE_OK;
}

// ---------------------------------------------------------------------------------------------
// Attention forward by per-branch linearisation.
//   q [N, hq, d], k/v [N, hkv, d] (fp64), kv head of q head h = h / (hq / hkv) (reading R10).
//   want [N] (nullable): only these rows are required.  check_invariant = 1 recomputes every
//   wanted row in every branch containing it and asserts BITWISE equality with the first write
//   (P:140); 0 computes each wanted row once (first branch in trajectory order).
//   o [N, hq, d], lse [hq, N] (natural log, reading R9).
// ---------------------------------------------------------------------------------------------
int oracle_attn_fwd(int64_t N, int32_t hq, int32_t hkv, int32_t d, double scale,
                    const double* q, const double* k, const double* v,
                    int64_t n_traj, const int64_t* path_ptr, const int32_t* path_idx,
                    const uint8_t* want, int32_t check_invariant,
                    double* o, double* lse, int32_t nthreads) {
  if (hq <= 0 || hkv <= 0 || hq % hkv || d <= 0) return OE_INVALID;
  const int g = hq / hkv;
  std::vector<int> bad(hq, 0);
  run_threads(hq, nthreads, [&](int h) {
    const int hk = h / g;
    std::vector<char> done(N, 0);
    std::vector<const double*> kr, vr;
    std::vector<double> s, orow(d);
    for (int64_t t = 0; t < n_traj; ++t) {
      const int32_t* idx = path_idx + path_ptr[t];
      const int64_t L = path_ptr[t + 1] - path_ptr[t];
      kr.resize(L); vr.resize(L);
      for (int64_t p = 0; p < L; ++p) {
        kr[p] = k + ((int64_t)idx[p] * hkv + hk) * d;
        vr[p] = v + ((int64_t)idx[p] * hkv + hk) * d;
      }
      for (int64_t p = 0; p < L; ++p) {
        const int64_t i = idx[p];
        if (want && !want[i]) continue;
        if (done[i] && !check_invariant) continue;
        double l;
        attn_row(q + (i * hq + h) * d, kr.data(), vr.data(), (int)(p + 1), d, scale, s, orow.data(), &l);
        double* out = o + (i * hq + h) * d;
        if (done[i]) {
          if (std::memcmp(out, orow.data(), d * 8) != 0 || std::memcmp(&lse[(int64_t)h * N + i], &l, 8) != 0)
            bad[h] = 1;
        } else {
          std::memcpy(out, orow.data(), d * 8);
          lse[(int64_t)h * N + i] = l;
          done[i] = 1;
        }
      }
    }
  });
  for (int h = 0; h < hq; ++h) if (bad[h]) return OE_INVARIANT;
  return OE_OK;
}

// ---------------------------------------------------------------------------------------------
// Attention backward by per-branch linearisation (Eqs. 2, 14-16, 20-21).
//   gup [N, hq, d]: upstream gradient G per packed token; every branch containing token i uses
//   dO_branch[p] = G[i] (the per-branch baseline gradient, Eq. 16 "dY^base").
//   Per branch, ordinary softmax-attention backward:
//     P_pj = exp(scale q_p.k_j - LSE_p),  D_p = G_p.O_p,  dS_pj = P_pj (G_p.v_j - D_p),
//     dQ_p += scale sum_j dS_pj k_j,  dK_j += scale dS_pj q_p,  dV_j += P_pj G_p.
//   Branch results are scatter-added into dq [N,hq,d], dk/dv [N,hkv,d] in ascending trajectory
//   order; dk/dv of a kv group are the sum over its q heads in ascending head order.
//   want_q / want_k (nullable [N]): rows whose dq / keys whose dk,dv are required.
//   traj_weight (nullable [n_traj]): objective sum_t alpha_t Loss_t (SPEC S:332 leaf_weights, S:475;
//   reading R20): branch t's gradients are multiplied by alpha_t before the scatter-add.
// ---------------------------------------------------------------------------------------------
int oracle_attn_bwd(int64_t N, int32_t hq, int32_t hkv, int32_t d, double scale,
                    const double* q, const double* k, const double* v, const double* gup,
                    int64_t n_traj, const int64_t* path_ptr, const int32_t* path_idx,
                    const double* traj_weight, const uint8_t* want_q, const uint8_t* want_k,
                    double* dq, double* dk, double* dv, int32_t nthreads) {
  if (hq <= 0 || hkv <= 0 || hq % hkv || d <= 0) return OE_INVALID;
  const int g = hq / hkv;
  const bool filt = want_q || want_k;
  std::vector<std::vector<double>> dk_h(hq), dv_h(hq);
  if (filt) {
    // Sampled mode: only the wanted outputs, each by the same arithmetic and in the same summation
    // order as the full mode below (bq[p] over keys j ascending; bk[j] / bv[j] over rows p
    // ascending within a branch; branches in trajectory order), so a wanted value is bitwise the
    // full mode's.  The work is split over rows (forward rows, dq rows) or keys (dk/dv), never
    // over the terms of one sum, so the result does not depend on the thread count.
    for (int64_t i = 0; i < N * hq * d; ++i) dq[i] = 0.0;
    std::vector<const double*> kr, vr;
    std::vector<double> O, LSE, Dv, bq, bk, bv;
    std::vector<int64_t> rows_q, keys;
    for (int h = 0; h < hq; ++h) {
      const int hk = h / g;
      dk_h[h].assign((size_t)N * d, 0.0);
      dv_h[h].assign((size_t)N * d, 0.0);
      for (int64_t t = 0; t < n_traj; ++t) {
        const int32_t* idx = path_idx + path_ptr[t];
        const int64_t L = path_ptr[t + 1] - path_ptr[t];
        if (L == 0) continue;
        int64_t p_min = L;
        if (want_k) {
          for (int64_t p = 0; p < L; ++p) if (want_k[idx[p]]) { p_min = p; break; }
        }
        rows_q.clear(); keys.clear();
        std::vector<char> need(L, 0);
        for (int64_t p = 0; p < L; ++p) {
          const bool wq = want_q && want_q[idx[p]];
          need[p] = wq || p >= p_min;
          if (wq) rows_q.push_back(p);
          if (want_k && want_k[idx[p]]) keys.push_back(p);
        }
        kr.resize(L); vr.resize(L);
        for (int64_t p = 0; p < L; ++p) {
          kr[p] = k + ((int64_t)idx[p] * hkv + hk) * d;
          vr[p] = v + ((int64_t)idx[p] * hkv + hk) * d;
        }
        O.assign((size_t)L * d, 0.0); LSE.assign(L, 0.0); Dv.assign(L, 0.0);
        bq.assign((size_t)L * d, 0.0); bk.assign((size_t)L * d, 0.0); bv.assign((size_t)L * d, 0.0);
        // forward rows + D_p (same arithmetic as the full mode)
        run_threads((int)L, nthreads, [&](int p) {
          if (!need[p]) return;
          std::vector<double> s;
          const double* gp = gup + ((int64_t)idx[p] * hq + h) * d;
          attn_row(q + ((int64_t)idx[p] * hq + h) * d, kr.data(), vr.data(), p + 1, d, scale, s, &O[(size_t)p * d],
                   &LSE[p]);
          double D = 0.0;
          for (int c = 0; c < d; ++c) D += gp[c] * O[(size_t)p * d + c];
          Dv[p] = D;
        });
        // dq of the wanted rows: sum over keys j <= p ascending
        run_threads((int)rows_q.size(), nthreads, [&](int r) {
          const int64_t p = rows_q[r];
          const double* qp = q + ((int64_t)idx[p] * hq + h) * d;
          const double* gp = gup + ((int64_t)idx[p] * hq + h) * d;
          for (int64_t j = 0; j <= p; ++j) {
            double acc = 0.0;
            for (int c = 0; c < d; ++c) acc += qp[c] * kr[j][c];
            double P = std::exp(scale * acc - LSE[p]);
            double dP = 0.0;
            for (int c = 0; c < d; ++c) dP += gp[c] * vr[j][c];
            double dS = P * (dP - Dv[p]);
            for (int c = 0; c < d; ++c) bq[p * d + c] += scale * dS * kr[j][c];
          }
        });
        // dk / dv of the wanted keys: sum over rows p >= j ascending
        run_threads((int)keys.size(), nthreads, [&](int r) {
          const int64_t j = keys[r];
          for (int64_t p = j; p < L; ++p) {
            const double* qp = q + ((int64_t)idx[p] * hq + h) * d;
            const double* gp = gup + ((int64_t)idx[p] * hq + h) * d;
            double acc = 0.0;
            for (int c = 0; c < d; ++c) acc += qp[c] * kr[j][c];
            double P = std::exp(scale * acc - LSE[p]);
            double dP = 0.0;
            for (int c = 0; c < d; ++c) dP += gp[c] * vr[j][c];
            double dS = P * (dP - Dv[p]);
            for (int c = 0; c < d; ++c) {
              bk[j * d + c] += scale * dS * qp[c];
              bv[j * d + c] += P * gp[c];
            }
          }
        });
        const double a = traj_weight ? traj_weight[t] : 1.0;
        for (int64_t p = 0; p < L; ++p) {
          const int64_t i = idx[p];
          for (int c = 0; c < d; ++c) {
            dq[(i * hq + h) * d + c] += a * bq[p * d + c];
            dk_h[h][i * d + c] += a * bk[p * d + c];
            dv_h[h][i * d + c] += a * bv[p * d + c];
          }
        }
      }
    }
  } else
  run_threads(hq, nthreads, [&](int h) {
    const int hk = h / g;
    dk_h[h].assign((size_t)N * d, 0.0);
    dv_h[h].assign((size_t)N * d, 0.0);
    for (int64_t i = 0; i < N; ++i)
      for (int c = 0; c < d; ++c) dq[(i * hq + h) * d + c] = 0.0;
    std::vector<const double*> kr, vr;
    std::vector<double> s, O, LSE, bq, bk, bv;
    for (int64_t t = 0; t < n_traj; ++t) {
      const int32_t* idx = path_idx + path_ptr[t];
      const int64_t L = path_ptr[t + 1] - path_ptr[t];
      if (L == 0) continue;
      // rows of this branch that must be processed
      int64_t p_min = L;
      if (want_k) {
        for (int64_t p = 0; p < L; ++p) if (want_k[idx[p]]) { p_min = p; break; }
      }
      std::vector<char> need(L, filt ? 0 : 1);
      if (filt) {
        for (int64_t p = 0; p < L; ++p)
          need[p] = (want_q && want_q[idx[p]]) || p >= p_min;
      }
      kr.resize(L); vr.resize(L);
      for (int64_t p = 0; p < L; ++p) {
        kr[p] = k + ((int64_t)idx[p] * hkv + hk) * d;
        vr[p] = v + ((int64_t)idx[p] * hkv + hk) * d;
      }
      O.assign((size_t)L * d, 0.0); LSE.assign(L, 0.0);
      bq.assign((size_t)L * d, 0.0); bk.assign((size_t)L * d, 0.0); bv.assign((size_t)L * d, 0.0);
      // forward rows (same arithmetic as oracle_attn_fwd)
      for (int64_t p = 0; p < L; ++p) {
        if (!need[p]) continue;
        attn_row(q + ((int64_t)idx[p] * hq + h) * d, kr.data(), vr.data(), (int)(p + 1), d, scale, s,
                 &O[p * d], &LSE[p]);
      }
      // backward rows
      for (int64_t p = 0; p < L; ++p) {
        if (!need[p]) continue;
        const double* qp = q + ((int64_t)idx[p] * hq + h) * d;
        const double* gp = gup + ((int64_t)idx[p] * hq + h) * d;
        double D = 0.0;
        for (int c = 0; c < d; ++c) D += gp[c] * O[p * d + c];
        for (int64_t j = 0; j <= p; ++j) {
          double acc = 0.0;
          for (int c = 0; c < d; ++c) acc += qp[c] * kr[j][c];
          double P = std::exp(scale * acc - LSE[p]);
          double dP = 0.0;
          for (int c = 0; c < d; ++c) dP += gp[c] * vr[j][c];
          double dS = P * (dP - D);
          for (int c = 0; c < d; ++c) {
            bq[p * d + c] += scale * dS * kr[j][c];
            bk[j * d + c] += scale * dS * qp[c];
            bv[j * d + c] += P * gp[c];
          }
        }
      }
      // scatter-add branch gradients into the tree arrays (Eq. 16: prefix grads are sums)
      const double a = traj_weight ? traj_weight[t] : 1.0;
      for (int64_t p = 0; p < L; ++p) {
        const int64_t i = idx[p];
        for (int c = 0; c < d; ++c) {
          dq[(i * hq + h) * d + c] += a * bq[p * d + c];
          dk_h[h][i * d + c] += a * bk[p * d + c];
          dv_h[h][i * d + c] += a * bv[p * d + c];
        }
      }
    }
  });
  for (int hk = 0; hk < hkv; ++hk) {
    for (int64_t i = 0; i < N; ++i)
      for (int c = 0; c < d; ++c) {
        double sk = 0.0, sv = 0.0;
        for (int r = 0; r < g; ++r) {
          sk += dk_h[hk * g + r][i * d + c];
          sv += dv_h[hk * g + r][i * d + c];
        }
        dk[(i * hkv + hk) * d + c] = sk;
        dv[(i * hkv + hk) * d + c] = sv;
      }
  }
  return OE_OK;
}

// ---------------------------------------------------------------------------------------------
// Next-token cross entropy by per-branch linearisation (readings R7, R8, R17).
//   Branch t has packed path idx[0..L).  For p < L-1 the token idx[p] predicts tok[idx[p+1]];
//   the prediction counts iff target_sup (nullable [N], per TARGET token) is set, and, when
//   boundary_mode == 1, iff every branch through idx[p] that continues continues to the same
//   packed token (SPEC S:375 exclusion at diverging branch points).
//   Only rows listed in row_ids are evaluated; x_rows[r, :] are the logits of row_ids[r].
//   Outputs per listed row: loss_rows (sum over branches of lse - x[target]), omega_rows (number
//   of counted predictions), dx_rows = gamma * sum over counted predictions (softmax - onehot).
//   traj_weight (nullable [n_traj]): each prediction of branch t counts alpha_t times (loss, omega
//   and dx), the objective sum_t alpha_t Loss_t of SPEC S:332 / S:475 (reading R20).
// ---------------------------------------------------------------------------------------------
int oracle_loss(int64_t N, int32_t V, const int32_t* tok, int64_t n_traj, const int64_t* path_ptr,
                const int32_t* path_idx, const double* traj_weight, const uint8_t* target_sup, int32_t boundary_mode, double gamma,
                int64_t n_rows, const int64_t* row_ids, const double* x_rows,
                double* loss_rows, double* omega_rows, double* dx_rows, int32_t nthreads) {
  if (V <= 0 || n_rows < 0) return OE_INVALID;
  std::vector<int64_t> slot(N, -1);
  for (int64_t r = 0; r < n_rows; ++r) {
    if (row_ids[r] < 0 || row_ids[r] >= N) return OE_INVALID;
    slot[row_ids[r]] = r;
  }
  // successor sets (for boundary_mode 1): next packed index per (token, branch)
  std::vector<int64_t> first_next(N, -1);
  std::vector<char> diverge(N, 0);
  for (int64_t t = 0; t < n_traj; ++t) {
    const int32_t* idx = path_idx + path_ptr[t];
    const int64_t L = path_ptr[t + 1] - path_ptr[t];
    for (int64_t p = 0; p + 1 < L; ++p) {
      int64_t i = idx[p], nx = idx[p + 1];
      if (first_next[i] < 0) first_next[i] = nx;
      else if (first_next[i] != nx) diverge[i] = 1;
    }
  }
  // occurrences (branch order) of every requested row
  std::vector<std::vector<std::pair<int64_t, double>>> occ_next(n_rows);
  for (int64_t t = 0; t < n_traj; ++t) {
    const int32_t* idx = path_idx + path_ptr[t];
    const int64_t L = path_ptr[t + 1] - path_ptr[t];
    const double a = traj_weight ? traj_weight[t] : 1.0;
    for (int64_t p = 0; p + 1 < L; ++p) {
      int64_t r = slot[idx[p]];
      if (r >= 0) occ_next[r].push_back({idx[p + 1], a});
    }
  }
  for (int64_t i = 0; i < N; ++i)
    if (tok[i] < 0 || tok[i] >= V) return OE_INVALID;
  run_threads((int)std::min<int64_t>(n_rows, INT32_MAX), nthreads, [&](int r) {
    const double* x = x_rows + (int64_t)r * V;
    double* dx = dx_rows + (int64_t)r * V;
    for (int32_t c = 0; c < V; ++c) dx[c] = 0.0;
    double loss = 0.0, omega = 0.0;
    const int64_t i = row_ids[r];
    for (const auto& oc : occ_next[r]) {
      const int64_t nx = oc.first;
      const double a = oc.second;
      if (target_sup && !target_sup[nx]) continue;
      if (boundary_mode == 1 && diverge[i]) continue;
      double m = -INFINITY;
      for (int32_t c = 0; c < V; ++c) m = std::max(m, x[c]);
      double l = 0.0;
      for (int32_t c = 0; c < V; ++c) l += std::exp(x[c] - m);
      double lse = m + std::log(l);
      int32_t y = tok[nx];
      loss += a * (lse - x[y]);
      omega += a;
      for (int32_t c = 0; c < V; ++c) dx[c] += gamma * a * std::exp(x[c] - lse);
      dx[y] -= gamma * a;
    }
    loss_rows[r] = loss;
    omega_rows[r] = omega;
  });
  return OE_OK;
}

}  // extern "C"
