"""Pins for the oracle's pack (oracle.cpp `oracle_pack`, `oracle_dense_mask`, `oracle_tiles`).

Pinned against: paper-printed tree-scales (Fig. 4gradient), SPEC worked examples
(S:73-97), closed-form accounting identities, brute-force
path enumeration, and the parent-walk mask definition (SPEC).
"""
import json
import os

import numpy as np
import pytest

import oracle
from workloads import trees

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _brute_paths(parent, length, term=None):
    """Independent path enumeration: every trajectory's node list, by parent walk."""
    n = len(parent)
    has_child = [False] * n
    for v in range(n):
        if parent[v] >= 0:
            has_child[parent[v]] = True
    term = term if term is not None else [0 if has_child[v] else 1 for v in range(n)]
    out = []
    for v in range(n):
        for _ in range(int(term[v])):
            nodes = []
            u = v
            while u >= 0:
                nodes.append(u)
                u = parent[u]
            out.append(nodes[::-1])
    return out


def test_fig4_paper_scales():
    g = json.load(open(os.path.join(GOLD, "fig4_gradient.json")))
    pk = oracle.pack(g["parent"], g["length"])
    names = g["node_names"]
    for nm, sc in g["paper_scale"].items():
        assert pk["node_leaves"][names.index(nm)] == sc, nm
    # per-token scale of the single token of r, u, v1
    assert pk["w"][pk["node_start"][names.index("r")]] == 5
    assert pk["w"][pk["node_start"][names.index("v1")]] == 3
    # full arrays (DFS pre-order, children ascending): hand-derived in SURVEY §8(c)
    assert pk["w"].tolist() == [5, 5, 3, 1, 1, 1, 2, 1, 1]
    assert pk["pos"].tolist() == [0, 1, 2, 3, 3, 3, 2, 3, 3]
    assert pk["E"].tolist() == [9, 9, 6, 4, 5, 6, 9, 8, 9]


def test_spec_example():
    g = json.load(open(os.path.join(GOLD, "spec_examples.json")))
    pk = oracle.pack(g["tree"]["parent"], g["tree"]["length"])
    assert pk["n_tokens"] == g["n_tokens"]
    assert int(pk["w"].sum()) == g["linear_tokens"]          # scale conservation, S:371 / S:80
    assert int(np.asarray(g["tree"]["length"]).sum()) == g["tree_tokens"]
    leaf_b = pk["node_start"][2]
    assert pk["pos"][leaf_b:leaf_b + 4].tolist() == g["leaf_b_pos"]
    assert pk["w"][0] == g["root_scale"]
    m = oracle.dense_mask(pk)
    a0, a1 = pk["node_start"][1], pk["node_sub_end"][1]
    b0, b1 = pk["node_start"][2], pk["node_sub_end"][2]
    assert not m[b0:b1, a0:a1].any()                            # leaf b cannot attend leaf a
    assert pk["pos"].tolist() == [0, 1, 2, 3, 4, 5, 6, 7, 5, 6, 7, 8]
    assert pk["E"].tolist() == [12] * 5 + [8] * 3 + [12] * 4


def test_tiny_config():
    pk = oracle.pack(*[np.asarray(x) for x in ([-1, 0, 0], [16, 8, 8])])
    assert pk["pos"].tolist() == list(range(16)) + list(range(16, 24)) * 2
    assert pk["w"].tolist() == [2] * 16 + [1] * 16
    assert pk["E"].tolist() == [32] * 16 + [24] * 8 + [32] * 8
    pos, w = pk["pos"].astype(np.int64), pk["w"].astype(np.int64)
    assert int((pos + 1).sum()) == 464                   # A
    assert int((w * (pos + 1)).sum()) == 600             # A_lin


def test_single_leaf_degenerates_to_causal():
    pk = oracle.pack([-1], [7])
    assert pk["pos"].tolist() == list(range(7))
    assert pk["w"].tolist() == [1] * 7
    m = oracle.dense_mask(pk)
    assert (m == np.tril(np.ones((7, 7), bool))).all()


def test_chain_is_lower_triangular():
    t = trees.chain(5, seg=3)
    pk = oracle.pack(t.parent, t.length)
    m = oracle.dense_mask(pk)
    assert (m == np.tril(np.ones((15, 15), bool))).all()
    assert pk["pos"].tolist() == list(range(15))


@pytest.mark.parametrize("seed", range(40))
def test_random_forest_invariants(seed):
    rng = np.random.default_rng(seed)
    t = trees.gen_random_forest(rng, max_nodes=14, max_len=6, with_term=(seed % 3 == 0))
    pk = oracle.pack(t.parent, t.length, t.term)
    N = pk["n_tokens"]
    assert N == int(t.length.sum())
    pos = pk["pos"].astype(np.int64)
    w = pk["w"].astype(np.int64)
    E = pk["E"]
    # brute-force paths (node lists) -> packed index lists must match the oracle's CSR
    bp = _brute_paths(t.parent.tolist(), t.length.tolist(), None if t.term is None else t.term.tolist())
    ops = oracle.paths(pk)
    assert len(bp) == len(ops)
    exp_paths = []
    for nodes in bp:
        exp = []
        for u in nodes:
            s = pk["node_start"][u]
            exp.extend(range(s, s + t.length[u]))
        exp_paths.append(tuple(exp))
    # same multiset of trajectories (the oracle orders them by DFS pre-order of the end node)
    assert sorted(exp_paths) == sorted(tuple(int(x) for x in idx) for idx in ops)
    for idx in ops:
        # path restriction gives positions 0..L-1
        assert pos[idx].tolist() == list(range(len(idx)))
    Ls = np.array([len(x) for x in ops], dtype=np.int64)
    # scale conservation: sum_i w_i = sum_l L_l
    assert int(w.sum()) == int(Ls.sum())
    # pair identity: sum_i w_i (pos_i + 1) = sum_l L_l (L_l + 1) / 2
    assert int((w * (pos + 1)).sum()) == int((Ls * (Ls + 1) // 2).sum())
    # w_i = number of trajectories through token i (brute force count)
    cnt = np.zeros(N, np.int64)
    for idx in ops:
        cnt[idx] += 1
    assert (cnt == w).all()
    # mask definition (parent walk) == interval form j <= i < E_j
    m = oracle.dense_mask(pk)
    ii, jj = np.meshgrid(np.arange(N), np.arange(N), indexing="ij")
    assert (m == ((jj <= ii) & (ii < E[jj]))).all()
    # DFS pre-order: each subtree occupies [start, sub_end)
    for u in range(t.n_nodes):
        s, e = pk["node_start"][u], pk["node_sub_end"][u]
        assert (pk["node"][s:s + t.length[u]] == u).all()
        sub = set()
        st = [u]
        while st:
            x = st.pop()
            sub.add(x)
            st.extend(np.flatnonzero(t.parent == x).tolist())
        assert set(pk["node"][s:e].tolist()) <= sub
        assert sum(int(t.length[x]) for x in sub) == e - s


@pytest.mark.parametrize("bad,err", [
    (([-1, 2, 1], [1, 1, 1]), 2),       # cycle 1 <-> 2
    (([0], [1]), 2),                    # self-parent
    (([-1, 5], [1, 1]), 2),             # parent out of range
    (([-1, -2], [1, 1]), 2),
    (([-1, 0], [0, 0]), 3),             # no tokens
    (([-1, 0], [1, -1]), 1),            # negative length
])
def test_pack_errors(bad, err):
    with pytest.raises(oracle.OracleError) as ei:
        oracle.pack(*bad)
    assert ei.value.code == err


def test_zero_length_and_multiroot():
    # root 0 (len 0) -> {1 (len 2), 2 (len 0) -> {3 (len 1)}}, plus a second root 4 (len 3)
    parent = [-1, 0, 0, 2, -1]
    length = [0, 2, 0, 1, 3]
    pk = oracle.pack(parent, length)
    assert pk["n_tokens"] == 6
    assert pk["pos"].tolist() == [0, 1, 0, 0, 1, 2]
    assert pk["w"].tolist() == [1, 1, 1, 1, 1, 1]
    assert pk["E"].tolist() == [2, 2, 3, 6, 6, 6]


def test_term_counts_duplicates_and_internal_ends():
    # trajectory ending at internal node 0 (term 1) + two identical trajectories ending at leaf 1
    pk = oracle.pack([-1, 0], [2, 2], [1, 2])
    assert pk["n_traj"] == 3
    assert pk["w"].tolist() == [3, 3, 2, 2]


def test_tiles_brute_force_vs_interval_rule():
    """Brute-force tile classes == the closed form of SURVEY App. A (empty iff maxE_kb <= i0,
    full iff minE_kb >= i1 off the diagonal) on agentic and wide trees."""
    for t, B in ((trees.gen_agentic(2048, root_len=256, seed=0), 64),
                 (trees.gen_wide(prefix=512, n_leaves=8), 64),
                 (trees.spec_example(), 4), (trees.fig4_unit(), 2)):
        pk = oracle.pack(t.parent, t.length)
        cls, mn, mx = oracle.tiles(pk, B)
        N = pk["n_tokens"]
        nb = (N + B - 1) // B
        for qb in range(nb):
            i0, i1 = qb * B, min(N, qb * B + B)
            for kb in range(nb):
                if kb > qb:
                    exp = 0
                elif kb == qb:
                    exp = 2 if (i1 - i0) == 1 else 1
                else:
                    exp = 0 if mx[kb] <= i0 else (2 if mn[kb] >= i1 else 1)
                assert cls[qb, kb] == exp, (t.name, qb, kb)
        # backward q-range per k-block is contiguous [kb, ceil(maxE/B))
        for kb in range(nb):
            nz = np.flatnonzero(cls[:, kb])
            assert nz.tolist() == list(range(kb, (mx[kb] + B - 1) // B))
