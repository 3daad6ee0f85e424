"""NEXT-f1 capacity-constrained Tree Packing: oracle pins (SPEC worked examples, brute force) and the
libtt host planner (validity + sandwich property) — all CPU."""
import time

import numpy as np
import pytest

from oracle import plan as P
from workloads import trees


# ---------------------------------------------------------------- oracle pins
def test_spec_feasibility_and_single_path_examples():
    # root(l=5), leaves (3, 4)
    par, ln = [-1, 0, 0], [5, 3, 4]
    L, nl, R = P.annotate(par, ln)
    assert (L[0], nl[0], R[0]) == (5, 2, 7)
    assert P.feasible(0, L, R, 12) and not P.feasible(0, L, R, 11)
    assert P.single_path_dp(par, ln, 12) == (5, [0])
    assert P.single_path_dp(par, ln, 11)[0] == 0
    # chain r(2) -> u(2) -> {v1(1), v2(1)}, C = 7 -> savings 4, selected {u}
    par, ln = [-1, 0, 1, 1], [2, 2, 1, 1]
    assert P.single_path_dp(par, ln, 7) == (4, [1])


def test_spec_multi_path_examples():
    # one traversal of cost 12 at C = 12; {a},{b} = 8 + 9 = 17 at C = 9
    assert P.brute_force_opt([-1, 0, 0], [5, 3, 4], 12) == 12
    assert P.brute_force_opt([-1, 0, 0], [5, 3, 4], 9) == 17


def test_fig3_multi_path_beats_single_path():
    # Fig. tree_pack_img: r -> u -> {v1, v5}; packing r->u->v1 and r->u->v5 separately
    # pays r, u twice; one traversal covering both pays them once when it fits
    par = [-1, 0, 1, 1, 2, 2, 3, 3]
    ln = [4, 4, 3, 3, 2, 2, 2, 2]
    C = 22
    sp_sav, _ = P.single_path_dp(par, ln, C)
    lin = P.linear_tokens(par, ln)
    opt = P.brute_force_opt(par, ln, C)
    assert opt < lin - sp_sav
    assert opt >= P.tree_tokens(par, ln)


@pytest.mark.parametrize("seed", range(25))
def test_single_path_dp_equals_antichain_brute_force(seed):
    rng = np.random.default_rng(seed)
    t = trees.gen_random_forest(rng, max_nodes=10, max_len=6, allow_zero=False, multi_root=False)
    L, nl, R = P.annotate(t.parent, t.length)
    C = int(max(L) + rng.integers(0, 12))
    sav, sel = P.single_path_dp(t.parent, t.length, C)
    assert sav == P.antichain_max(t.parent, t.length, C)


@pytest.mark.parametrize("seed", range(20))
def test_brute_force_sandwich_and_monotone(seed):
    rng = np.random.default_rng(100 + seed)
    t = trees.gen_random_forest(rng, max_nodes=9, max_len=6, allow_zero=False, multi_root=False)
    trajs = P.trajectories(t.parent, t.length)
    if len(trajs) > 7:
        pytest.skip("too many trajectories for exhaustive search")
    lin, tree_tok = P.linear_tokens(t.parent, t.length), P.tree_tokens(t.parent, t.length)
    Lmax = max(P.traversal_cost(t.parent, t.length, [p]) for p in trajs)
    prev = None
    for C in range(Lmax, tree_tok + 2):
        opt = P.brute_force_opt(t.parent, t.length, C)
        sp = lin - P.single_path_dp(t.parent, t.length, C)[0]
        assert tree_tok <= opt <= sp <= lin
        assert (opt == tree_tok) == (C >= tree_tok)
        if prev is not None:
            assert opt <= prev  # more capacity never costs more
        prev = opt


# ---------------------------------------------------------------- libtt planner
@pytest.fixture(scope="module")
def tt():
    from paper_2511_00413_b200 import build
    build.build()
    import paper_2511_00413_b200 as T
    T.lib()
    return T


@pytest.mark.parametrize("seed", range(40))
def test_planner_valid_and_sandwiched(tt, seed):
    rng = np.random.default_rng(500 + seed)
    t = trees.gen_random_forest(rng, max_nodes=9, max_len=7, with_term=(seed % 4 == 0))
    trajs = P.trajectories(t.parent, t.length, t.term)
    if not trajs:
        pytest.skip("no trajectories")
    Lmax = max(P.traversal_cost(t.parent, t.length, [p]) for p in trajs)
    tree_tok = P.tree_tokens(t.parent, t.length, t.term)
    lin = P.linear_tokens(t.parent, t.length, t.term)
    for C in sorted({max(Lmax, 1), Lmax + 3, (Lmax + tree_tok) // 2, tree_tok, tree_tok + 5}):
        C = max(C, Lmax, 1)
        a, info = tt.tt_plan_traversals(t.parent, t.length, C, t.term)
        ok, costs = P.validate_plan(t.parent, t.length, C, a, t.term)
        assert ok, (C, a, costs)
        assert info["planned_tokens"] == sum(costs)
        assert info["linear_tokens"] == lin and info["tree_tokens"] == tree_tok
        assert info["n_traversals"] == len(costs)
        if len(trajs) <= 7:
            assert P.brute_force_opt(t.parent, t.length, C, t.term) <= info["planned_tokens"]
        assert info["planned_tokens"] <= lin
        if C >= tree_tok:
            assert info["n_traversals"] == 1 and info["planned_tokens"] == tree_tok


def test_planner_infeasible_trajectory(tt):
    with pytest.raises(tt.TTError) as ei:
        tt.tt_plan_traversals([-1, 0], [5, 6], 10)
    assert ei.value.code == 4


def test_traversal_forest_packs_to_its_cost(tt):
    t = trees.gen_agentic(3000, root_len=400, seed=6)
    C = 1600
    a, info = tt.tt_plan_traversals(t.parent, t.length, C)
    trajs = P.trajectories(t.parent, t.length)
    total, lin = 0, 0
    for k in range(info["n_traversals"]):
        par, ln, term, old = tt.tt_traversal_forest(t.parent, t.length, a, k)
        pi = tt.tt_pack_plan(par, ln, term)
        grp = [trajs[i] for i in np.flatnonzero(a == k)]
        assert pi["n_tokens"] == P.traversal_cost(t.parent, t.length, grp) <= C
        assert pi["n_traj"] == len(grp)
        # in-traversal tree-scale: sum_i w_i = sum of the traversal's path lengths
        assert pi["n_linear_tokens"] == sum(P.traversal_cost(t.parent, t.length, [p]) for p in grp)
        total += pi["n_tokens"]
        lin += pi["n_linear_tokens"]
    assert total == info["planned_tokens"] and lin == info["linear_tokens"]


def test_planner_scales(tt):
    """10^5-node forest (deep chains + wide fans) plans in well under a second."""
    rng = np.random.default_rng(0)
    n = 100_000
    parent = np.empty(n, np.int64)
    parent[0] = -1
    for v in range(1, n):
        parent[v] = v - 1 if rng.random() < 0.3 else int(rng.integers(0, v))
    length = rng.integers(1, 40, n)
    t0 = time.perf_counter()
    a, info = tt.tt_plan_traversals(parent, length, 1 << 22)
    dt = time.perf_counter() - t0
    assert dt < 2.0
    assert info["planned_tokens"] <= info["linear_tokens"]
    assert info["planned_tokens"] >= info["tree_tokens"]
