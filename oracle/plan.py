"""Capacity-constrained Tree Packing references — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Plain, slow, definition-level Python for SURVEY §8(f) NEXT-f1 (§2.2):

  annotate(...)        L(u), n_u, R(u) of P:174-179 (SPEC S:47-54 endpoint convention: L includes u's
                       own segment, d(u, l) excludes it)
  feasible(...)        Eq. 3: L(u) + R(u) <= C
  single_path_dp(...)  Eq. 5: DP(u) = max(1_f(u) (n_u - 1) L(u), sum_children DP(v)), DP(leaf)=0;
                       single-path cost = linear tokens - DP(roots)
  antichain_max(...)   brute force over antichains of shared nodes (pins single_path_dp)
  traversal_cost(...)  tokens of the sub-forest induced by a set of trajectories
  brute_force_opt(...) the optimum the multi-path DP (Eqs. 6-11) computes, by its
                       definition: minimum total traversal cost over all partitions of the
                       trajectories into traversals of cost <= C (exhaustive; tiny trees only)

Trajectories are numbered in canonical order (DFS pre-order of end nodes, roots / children ascending
id, term copies consecutive) — the order oracle.pack uses.
"""
from __future__ import annotations

from itertools import combinations
from typing import List, Sequence

import numpy as np


def _children(parent):
    n = len(parent)
    kids = [[] for _ in range(n)]
    roots = []
    for v in range(n):
        (roots if parent[v] < 0 else kids[parent[v]]).append(v)
    return kids, roots


def trajectories(parent, length, term=None) -> List[List[int]]:
    """Canonical trajectories as root-to-end node lists."""
    parent = list(map(int, parent))
    kids, roots = _children(parent)
    n = len(parent)
    if term is None:
        term = [0 if kids[v] else 1 for v in range(n)]
    out = []

    def visit(u, path):
        path = path + [u]
        for _ in range(int(term[u])):
            out.append(path)
        for c in kids[u]:
            visit(c, path)

    for r in roots:
        visit(r, [])
    return out


def annotate(parent, length):
    """L(u) (inclusive prefix length), n_u (leaves under u), R(u) = sum over leaves of d(u, leaf)
    with d excluding u's own segment.  Leaf-terminated trees (default term)."""
    parent = list(map(int, parent))
    length = list(map(int, length))
    kids, roots = _children(parent)
    n = len(parent)
    L = [0] * n
    nl = [0] * n
    R = [0] * n

    def down(u, acc):
        L[u] = acc + length[u]
        for c in kids[u]:
            down(c, L[u])

    def up(u):
        if not kids[u]:
            nl[u], R[u] = 1, 0
            return
        for c in kids[u]:
            up(c)
        nl[u] = sum(nl[c] for c in kids[u])
        R[u] = sum(nl[c] * length[c] + R[c] for c in kids[u])

    for r in roots:
        down(r, 0)
        up(r)
    return L, nl, R


def feasible(u, L, R, C) -> bool:
    return L[u] + R[u] <= C


def single_path_dp(parent, length, C):
    """Eq. 5.  Returns (savings, selected antichain).  Requires every leaf path <= C."""
    parent = list(map(int, parent))
    kids, roots = _children(parent)
    L, nl, R = annotate(parent, length)
    for u in range(len(parent)):
        if not kids[u] and L[u] > C:
            raise ValueError("a leaf does not fit the capacity")
    best = {}

    def dp(u):
        if not kids[u]:
            best[u] = (0, [u])
            return 0
        child_sum = sum(dp(c) for c in kids[u])
        share = (nl[u] - 1) * L[u] if feasible(u, L, R, C) else 0
        if feasible(u, L, R, C) and share >= child_sum:
            best[u] = (share, [u])
        else:
            best[u] = (child_sum, [x for c in kids[u] for x in best[c][1]])
        return best[u][0]

    total, sel = 0, []
    for r in roots:
        total += dp(r)
        sel += best[r][1]
    return total, sel


def antichain_max(parent, length, C) -> int:
    """Brute force over antichains whose subtrees partition the leaves (the single-path problem)."""
    parent = list(map(int, parent))
    kids, roots = _children(parent)
    L, nl, R = annotate(parent, length)
    n = len(parent)
    leaves = [v for v in range(n) if not kids[v]]

    def leafset(u):
        if not kids[u]:
            return {u}
        s = set()
        for c in kids[u]:
            s |= leafset(c)
        return s

    ls = [frozenset(leafset(u)) for u in range(n)]
    best = -1
    for k in range(1, n + 1):
        for combo in combinations(range(n), k):
            cover = set()
            ok = True
            for u in combo:
                if cover & ls[u]:
                    ok = False
                    break
                cover |= ls[u]
            if not ok or cover != set(leaves):
                continue
            sav = 0
            for u in combo:
                if kids[u]:
                    if not feasible(u, L, R, C):
                        ok = False
                        break
                    sav += (nl[u] - 1) * L[u]
            if ok:
                best = max(best, sav)
    return best


def traversal_cost(parent, length, trajs: Sequence[Sequence[int]]) -> int:
    nodes = set()
    for path in trajs:
        nodes.update(path)
    return int(sum(int(length[u]) for u in nodes))


def _partitions(items):
    if not items:
        yield []
        return
    first, rest = items[0], items[1:]
    for part in _partitions(rest):
        for i in range(len(part)):
            yield part[:i] + [[first] + part[i]] + part[i + 1:]
        yield [[first]] + part


def brute_force_opt(parent, length, C, term=None) -> int:
    """Minimum total cost over all partitions of the trajectories into traversals of cost <= C
    (exhaustive; <= ~9 trajectories).  Returns -1 if infeasible."""
    trajs = trajectories(parent, length, term)
    best = -1
    for part in _partitions(list(range(len(trajs)))):
        tot = 0
        ok = True
        for grp in part:
            c = traversal_cost(parent, length, [trajs[k] for k in grp])
            if c > C:
                ok = False
                break
            tot += c
        if ok and (best < 0 or tot < best):
            best = tot
    return best


def linear_tokens(parent, length, term=None) -> int:
    return int(sum(traversal_cost(parent, length, [p]) for p in trajectories(parent, length, term)))


def tree_tokens(parent, length, term=None) -> int:
    return traversal_cost(parent, length, trajectories(parent, length, term))


def validate_plan(parent, length, C, traversal_of_traj, term=None):
    """Returns (ok, per-traversal costs).  ok iff every trajectory is in exactly one traversal and
    every traversal's induced cost <= C."""
    trajs = trajectories(parent, length, term)
    a = np.asarray(traversal_of_traj)
    if len(a) != len(trajs):
        return False, []
    costs = []
    for t in range(int(a.max()) + 1 if len(a) else 0):
        grp = [trajs[k] for k in np.flatnonzero(a == t)]
        if not grp:
            return False, costs
        costs.append(traversal_cost(parent, length, grp))
    return all(c <= C for c in costs), costs
