"""Pins for the oracle's real-valued leaf weights (NEXT-f4; SPEC S:332 leaf_weights, S:475
"non-uniform leaf weights ... scaler = weight sums"; reading R20: objective sum_l alpha_l Loss_l).

Pinned against:
  * brute force: dense masked attention over the packed sequence in torch fp64 whose autograd
    upstream gradient is W_i * G_i, W_i = sum of alpha over the trajectories through token i found
    by walking parent pointers (SURVEY App. B with w -> W, linear in Eq. 12);
  * a different mechanism: integer weights m_l give the same gradients and loss as repeating
    trajectory l m_l times through `term` (SPEC S:43-44 duplicate trajectories);
  * library special case: a one-hot weight on trajectory l equals torch SDPA(is_causal) autograd on
    the linearised branch l alone, scattered to its packed rows;
  * per-branch torch cross entropy weighted by alpha_l.
"""
import math

import numpy as np
import pytest
import torch

import oracle
from workloads import trees



@pytest.fixture(autouse=True, scope="module")
def _fp64_default():
    # fp64 default dtype for this module's tensors only (restored afterwards, so it cannot leak into
    # other modules' tensors, e.g. fp32 GPU outputs)
    prev = torch.get_default_dtype()
    torch.set_default_dtype(torch.float64)
    yield
    torch.set_default_dtype(prev)


def _rand(N, hq, hkv, d, seed):
    g = torch.Generator().manual_seed(seed)
    return [torch.randn(N, h, d, generator=g, dtype=torch.float64) for h in (hq, hkv, hkv, hq)]


def _ancestor_mask(t, pk):
    """allowed(i, j) by walking parent pointers from node(i), independent of E."""
    N = pk["n_tokens"]
    node = pk["node"]
    par = list(map(int, t.parent))
    anc = []
    for u in range(len(par)):
        s, x = set(), u
        while x >= 0:
            s.add(x)
            x = par[x]
        anc.append(s)
    m = np.zeros((N, N), bool)
    pos = pk["pos"]
    for i in range(N):
        for j in range(i + 1):
            m[i, j] = node[j] in anc[node[i]] and pos[j] <= pos[i]
    return torch.tensor(m)


def _token_weight(t, pk, alpha):
    """W_i = sum of alpha_l over trajectories through token i, from parent walks of end nodes."""
    par = list(map(int, t.parent))
    n = len(par)
    kids = [[] for _ in range(n)]
    for v in range(n):
        if par[v] >= 0:
            kids[par[v]].append(v)
    term = t.term if t.term is not None else [0 if kids[v] else 1 for v in range(n)]
    # canonical order: DFS pre-order of end nodes, roots / children ascending id
    ends = []

    def visit(u):
        ends.extend([u] * int(term[u]))
        for c in kids[u]:
            visit(c)

    for r in range(n):
        if par[r] < 0:
            visit(r)
    Wn = np.zeros(n)
    for a, u in zip(alpha, ends):
        x = u
        while x >= 0:
            Wn[x] += a
            x = par[x]
    return torch.tensor(Wn[pk["node"]])


CASES = [trees.spec_example(), trees.fig4_unit(), trees.Tree([-1, 0, 0, 2, -1, 4, 4], [3, 4, 0, 2, 5, 1, 3]),
         trees.Tree([-1, 0, 0, 1], [4, 3, 2, 3], [0, 1, 2, 1])]


@pytest.mark.parametrize("t", CASES, ids=lambda t: t.name)
def test_weighted_bwd_equals_dense_autograd(t):
    pk = oracle.pack(t.parent, t.length, t.term)
    N = pk["n_tokens"]
    rng = np.random.default_rng(3)
    alpha = rng.normal(size=pk["n_traj"])  # RL-style advantages: any sign
    hq, hkv, d = 4, 2, 8
    q, k, v, G = _rand(N, hq, hkv, d, seed=N)
    scale = 1 / math.sqrt(d)
    mask = _ancestor_mask(t, pk)
    g = hq // hkv
    qt = q.clone().requires_grad_(True)
    kt = k.clone().requires_grad_(True)
    vt = v.clone().requires_grad_(True)
    kk = kt.repeat_interleave(g, 1)
    vv = vt.repeat_interleave(g, 1)
    S = torch.einsum("ihc,jhc->hij", qt, kk) * scale
    P = torch.softmax(S.masked_fill(~mask[None], float("-inf")), dim=-1)
    o = torch.einsum("hij,jhc->ihc", P, vv)
    W = _token_weight(t, pk, alpha)
    o.backward(W[:, None, None] * G)
    dq, dk, dv = oracle.attn_bwd(pk, q, k, v, G, scale, traj_weight=alpha)
    for a, b in ((dq, qt.grad), (dk, kt.grad), (dv, vt.grad)):
        assert np.allclose(a, b.numpy(), rtol=1e-10, atol=1e-11)


def test_integer_weights_equal_duplicated_trajectories():
    t = trees.Tree([-1, 0, 0, 1, 1], [5, 3, 4, 2, 3])  # leaves 2, 3, 4
    m = [2, 3, 1]  # canonical order: node 3, node 4, node 2 (pre-order of ends)
    term = np.zeros(5, np.int32)
    term[[3, 4, 2]] = m
    pk1 = oracle.pack(t.parent, t.length)
    pk2 = oracle.pack(t.parent, t.length, term)
    assert pk2["n_traj"] == 6 and np.array_equal(pk1["node"], pk2["node"])
    N = pk1["n_tokens"]
    q, k, v, G = _rand(N, 2, 1, 8, seed=5)
    g1 = oracle.attn_bwd(pk1, q, k, v, G, 0.3, traj_weight=np.array(m, float))
    g2 = oracle.attn_bwd(pk2, q, k, v, G, 0.3)
    for a, b in zip(g1, g2):
        assert np.allclose(a, b, rtol=1e-12, atol=1e-13)
    V = 19
    x = torch.randn(N, V, generator=torch.Generator().manual_seed(1))
    tok = torch.randint(0, V, (N,), generator=torch.Generator().manual_seed(2), dtype=torch.int32)
    l1 = oracle.loss(pk1, tok, V, np.arange(N), x, gamma=0.5, traj_weight=np.array(m, float))
    l2 = oracle.loss(pk2, tok, V, np.arange(N), x, gamma=0.5)
    for a, b in zip(l1, l2):
        assert np.allclose(a, b, rtol=1e-12, atol=1e-13)


@pytest.mark.parametrize("which", [0, 2, 4])
def test_one_hot_weight_equals_branch_sdpa(which):
    t = trees.fig4_unit()
    pk = oracle.pack(t.parent, t.length)
    N = pk["n_tokens"]
    hq, hkv, d = 2, 2, 16
    q, k, v, G = _rand(N, hq, hkv, d, seed=9)
    alpha = np.zeros(pk["n_traj"])
    if which >= pk["n_traj"]:
        pytest.skip("fewer trajectories")
    alpha[which] = 1.0
    dq, dk, dv = oracle.attn_bwd(pk, q, k, v, G, 0.25, traj_weight=alpha)
    idx = torch.tensor(oracle.paths(pk)[which], dtype=torch.long)
    qt = q[idx].transpose(0, 1).clone().requires_grad_(True)
    kt = k[idx].transpose(0, 1).clone().requires_grad_(True)
    vt = v[idx].transpose(0, 1).clone().requires_grad_(True)
    o = torch.nn.functional.scaled_dot_product_attention(qt, kt, vt, is_causal=True, scale=0.25)
    o.backward(G[idx].transpose(0, 1))
    ref = [torch.zeros(N, hq, d) for _ in range(3)]
    for r, gr in zip(ref, (qt.grad, kt.grad, vt.grad)):
        r[idx] = gr.transpose(0, 1)
    for a, b in zip((dq, dk, dv), ref):
        assert np.allclose(a, b.numpy(), rtol=1e-10, atol=1e-12)


@pytest.mark.parametrize("t", CASES, ids=lambda t: t.name)
def test_weighted_loss_equals_weighted_branch_ce(t):
    pk = oracle.pack(t.parent, t.length, t.term)
    N = pk["n_tokens"]
    V = 23
    gx = torch.Generator().manual_seed(4)
    x = torch.randn(N, V, generator=gx) * 2
    tok = torch.randint(0, V, (N,), generator=gx, dtype=torch.int32)
    alpha = np.random.default_rng(7).uniform(-1.5, 2.5, pk["n_traj"])
    xx = x.clone().requires_grad_(True)
    total = torch.zeros(())
    omega = np.zeros(N)
    for a, idx in zip(alpha, oracle.paths(pk)):
        if len(idx) < 2:
            continue
        src = torch.tensor(idx[:-1], dtype=torch.long)
        tgt = torch.tensor(idx[1:], dtype=torch.long)
        total = total + a * torch.nn.functional.cross_entropy(xx[src], tok[tgt].long(), reduction="sum")
        np.add.at(omega, src.numpy(), a)
    gamma = 0.8
    (gamma * total).backward()
    total = float(total.detach())
    lr, om, dx = oracle.loss(pk, tok, V, np.arange(N), x, gamma=gamma, traj_weight=alpha)
    assert abs(lr.sum() - total) <= 1e-11 * max(1.0, abs(total))
    assert np.allclose(om, omega, rtol=1e-12, atol=1e-12)
    assert np.allclose(dx, xx.grad.numpy(), rtol=1e-10, atol=1e-12)
