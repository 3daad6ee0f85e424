"""Seeded tree shapes: parent array + per-node token counts (SURVEY.md §8(d) "Synthetic inputs").

A tree (or forest) is given exactly as the C ABI takes it (include/tt.h, `tt_pack`):
  parent[n] : int32, -1 for a root, else the index of the parent node
  len[n]    : int32 >= 0, tokens in the node's segment (l(y))
  term[n]   : optional int32 >= 0, trajectories ending at the node (default: 1 on childless nodes)
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np


@dataclass
class Tree:
    parent: np.ndarray
    length: np.ndarray
    term: Optional[np.ndarray] = None
    name: str = "tree"
    meta: dict = field(default_factory=dict)

    def __post_init__(self):
        self.parent = np.ascontiguousarray(self.parent, dtype=np.int32)
        self.length = np.ascontiguousarray(self.length, dtype=np.int32)
        if self.term is not None:
            self.term = np.ascontiguousarray(self.term, dtype=np.int32)

    @property
    def n_nodes(self) -> int:
        return int(self.parent.shape[0])

    @property
    def n_tokens(self) -> int:
        return int(self.length.sum())


def tiny() -> Tree:
    """Config 1: 16-token root prefix + 2 leaf branches of 8 tokens (BASELINE.json configs[0])."""
    return Tree([-1, 0, 0], [16, 8, 8], name="tiny")


def spec_example() -> Tree:
    """root(l=5) with leaves a(l=3), b(l=4)."""
    return Tree([-1, 0, 0], [5, 3, 4], name="spec_5_3_4")


def fig4_unit() -> Tree:
    """Shape of PAPER.md Fig. `4gradient`: r -> u -> {v1, v5}; v1 -> 3 leaves;
    v5 -> 2 leaves; one token per node.  Node ids: r=0, u=1, v1=2, v5=3, leaves 4,5,6 under v1?

    We use the SURVEY §8(c) encoding parent=[-1,0,1,1,2,2,2,3,3]: nodes 4,5,6 are children of
    v1=2 and nodes 7,8 children of v5=3.
    """
    return Tree([-1, 0, 1, 1, 2, 2, 2, 3, 3], [1] * 9, name="fig4_unit")


def chain(n_nodes: int, seg: int = 1) -> Tree:
    return Tree([-1] + list(range(n_nodes - 1)), [seg] * n_nodes, name=f"chain{n_nodes}")


def star(prefix: int, leaves) -> Tree:
    leaves = list(leaves)
    return Tree([-1] + [0] * len(leaves), [prefix] + leaves, name=f"star{prefix}x{len(leaves)}")


def _split_lengths(rng, n_nonroot: int, total: int, sigma: float) -> np.ndarray:
    """Split `total` tokens over n_nonroot nodes proportional to lognormal(0, sigma) shares:
    floor, clamp to >= 1, then fix up by +1 / -1 in share order until the sum is exact."""
    raw = rng.lognormal(0.0, sigma, n_nonroot)
    frac = raw / raw.sum() * total
    out = np.maximum(np.floor(frac).astype(np.int64), 1)
    order = np.argsort(-frac, kind="stable")
    diff = int(total - out.sum())
    i = 0
    guard = 0
    while diff > 0:
        out[order[i % n_nonroot]] += 1
        diff -= 1
        i += 1
    rev = order[::-1]
    i = 0
    while diff < 0:
        k = rev[i % n_nonroot]
        if out[k] > 1:
            out[k] -= 1
            diff += 1
        i += 1
        guard += 1
        if guard > 10 * n_nonroot + 10 * total:
            raise ValueError("cannot split tokens: too few for the node count")
    return out


def _agentic_shape(rng, D: int, bmin: int, bmax: int, p_open: float):
    parent = [-1]
    frontier = [0]
    for lv in range(1, D):
        nxt = []
        for u in frontier:
            b = int(rng.integers(bmin, bmax + 1))
            kids = list(range(len(parent), len(parent) + b))
            parent.extend([u] * b)
            if lv + 1 < D:
                opens = [bool(rng.random() < p_open) for _ in kids]
                if not any(opens):
                    opens[0] = True
                nxt.extend(k for k, o in zip(kids, opens) if o)
        frontier = nxt
    return parent


def gen_agentic(N: int, D: int = 6, bmin: int = 2, bmax: int = 4, p_open: float = 0.5,
                root_len: int = 1024, sigma: float = 1.0, seed: int = 0) -> Tree:
    """SURVEY.md §8(d) prototype generator `gen_agentic` (re-implemented exactly as described):
    the root is level 1; for lv = 1..D-1, each frontier node (creation order) draws b ~ U{bmin..bmax}
    children; if lv+1 < D each child stays open with prob p_open (first child forced open if none).
    After all structure draws, the N - root_len remaining tokens are split over non-root nodes
    proportional to lognormal(0, sigma) shares."""
    rng = np.random.default_rng(seed)
    parent = _agentic_shape(rng, D, bmin, bmax, p_open)
    n = len(parent)
    lens = np.empty(n, dtype=np.int64)
    lens[0] = root_len
    lens[1:] = _split_lengths(rng, n - 1, N - root_len, sigma)
    return Tree(parent, lens, name=f"agentic{N}_s{seed}",
                meta=dict(N=N, D=D, p_open=p_open, root_len=root_len, seed=seed))


def path_token_total(tree: Tree) -> int:
    """Sum over trajectories of their root-to-end path length (the per-branch linear token count;
    SPEC.md S:75-77).  Plain parent walk; used only to pick generator parameters."""
    parent = tree.parent
    n = tree.n_nodes
    has_child = np.zeros(n, dtype=bool)
    for v in range(n):
        if parent[v] >= 0:
            has_child[parent[v]] = True
    term = tree.term if tree.term is not None else (~has_child).astype(np.int64)
    total = 0
    for v in range(n):
        if term[v] == 0:
            continue
        s, u = 0, v
        while u >= 0:
            s += int(tree.length[u])
            u = int(parent[u])
        total += int(term[v]) * s
    return total


def gen_deep(N: int = 32768, seed: int = 1, p_open: float = 0.2, lo: int = 4096, hi: int = 16384,
             grid: int = 64, target_ratio: float = 4.0) -> Tree:
    """Config 3 / 5 generator: gen_agentic(N, p_open=0.2) with root_len on a `grid`-token grid in
    [lo, hi] whose per-branch token ratio is closest to `target_ratio`."""
    best = None
    for root_len in range(lo, hi + 1, grid):
        t = gen_agentic(N, p_open=p_open, root_len=root_len, seed=seed)
        r = path_token_total(t) / N
        key = (abs(r - target_ratio), root_len)
        if best is None or key < best[0]:
            best = (key, t, r)
    t = best[1]
    t.name = f"deep{N}_s{seed}"
    t.meta["token_ratio"] = best[2]
    return t


def gen_wide(prefix: int = 4096, n_leaves: int = 64, aligned: bool = False, seed: int = 4) -> Tree:
    """Config 4: a 4K-token prefix fanning out to 64 short leaves (concurrent tool calls).
    Ragged leaf lengths default_rng(4).integers(64, 193, 64); aligned variant: all 128."""
    if aligned:
        leaves = [128] * n_leaves
    else:
        leaves = np.random.default_rng(seed).integers(64, 193, n_leaves).tolist()
    t = star(prefix, leaves)
    t.name = f"wide{prefix}x{n_leaves}{'_aligned' if aligned else ''}"
    return t


def gen_random_forest(rng: np.random.Generator, max_nodes: int = 12, max_len: int = 9,
                      allow_zero: bool = True, multi_root: bool = True, with_term: bool = False) -> Tree:
    """Small random forests for property tests: random parent < child ids, random lengths
    (zero-length nodes allowed), several roots, optional explicit term[] counts."""
    n = int(rng.integers(1, max_nodes + 1))
    parent = [-1]
    for v in range(1, n):
        if multi_root and rng.random() < 0.15:
            parent.append(-1)
        else:
            parent.append(int(rng.integers(0, v)))
    lo = 0 if allow_zero else 1
    lens = rng.integers(lo, max_len + 1, n)
    # ensure at least one token overall
    if lens.sum() == 0:
        lens[0] = 1
    term = None
    if with_term:
        has_child = np.zeros(n, dtype=bool)
        for v in range(n):
            if parent[v] >= 0:
                has_child[parent[v]] = True
        term = np.where(has_child, rng.integers(0, 2, n), rng.integers(0, 3, n)).astype(np.int32)
        if term.sum() == 0:
            term[int(np.flatnonzero(~has_child)[0])] = 1
    # relabel so that parent ids are arbitrary (not always < child): random permutation
    perm = rng.permutation(n)
    inv = np.empty(n, dtype=np.int64)
    inv[perm] = np.arange(n)
    new_parent = np.empty(n, dtype=np.int64)
    new_len = np.empty(n, dtype=np.int64)
    new_term = None if term is None else np.empty(n, dtype=np.int64)
    for v in range(n):
        nv = inv[v]
        new_parent[nv] = -1 if parent[v] < 0 else inv[parent[v]]
        new_len[nv] = lens[v]
        if term is not None:
            new_term[nv] = term[v]
    return Tree(new_parent, new_len, new_term, name="random")


# BASELINE.json configs -> (tree factory, Hq, Hkv, d, dtype)
CONFIGS = {
    "tiny": dict(tree=lambda seed=0: tiny(), hq=1, hkv=1, d=64, dtype="fp32"),
    "agentic8k": dict(tree=lambda seed=0: gen_agentic(8192, p_open=0.5, root_len=1024, seed=seed),
                      hq=32, hkv=32, d=128, dtype="bf16"),
    "deep32k": dict(tree=lambda seed=1: gen_deep(32768, seed=seed), hq=32, hkv=8, d=128, dtype="bf16"),
    "wide": dict(tree=lambda seed=4: gen_wide(), hq=32, hkv=8, d=128, dtype="bf16"),
    "wide_aligned": dict(tree=lambda seed=4: gen_wide(aligned=True), hq=32, hkv=8, d=128, dtype="bf16"),
    "batch64k": dict(tree=lambda seed=0: gen_deep(65536, seed=seed, lo=8192, hi=32768),
                     hq=32, hkv=8, d=128, dtype="bf16"),
}


def config_tree(name: str, seed: Optional[int] = None) -> Tree:
    c = CONFIGS[name]
    return c["tree"]() if seed is None else c["tree"](seed)
