"""Pins for the oracle's Gradient-Restoration loss (oracle.cpp `oracle_loss`).

Pinned against: torch.nn.functional.cross_entropy(reduction='sum') in fp64 run on every
linearised branch and summed (library special case; "total loss = sum_l CE(path l)"),
its autograd for the logits gradient, the uniform-logits closed form (CE = ln V), and the
accounting identity sum Omega = sum_l (L_l - 1).
"""
import math

import numpy as np
import pytest
import torch

import oracle
from workloads import trees


def _setup(t, V, seed):
    pk = oracle.pack(t.parent, t.length, t.term)
    N = pk["n_tokens"]
    g = torch.Generator().manual_seed(seed)
    x = torch.randn(N, V, generator=g, dtype=torch.float64) * 2
    tok = torch.randint(0, V, (N,), generator=g, dtype=torch.int32)
    return pk, N, x, tok


def _torch_branch_ce(pk, x, tok, gamma, sup=None):
    xx = x.clone().requires_grad_(True)
    total = torch.zeros((), dtype=torch.float64)
    omega = np.zeros(x.shape[0])
    for idx in oracle.paths(pk):
        if len(idx) < 2:
            continue
        src = torch.tensor(idx[:-1], dtype=torch.long)
        tgt = torch.tensor(idx[1:], dtype=torch.long)
        if sup is not None:
            keep = torch.tensor(sup[idx[1:]], dtype=torch.bool)
            src, tgt = src[keep], tgt[keep]
        if len(src) == 0:
            continue
        total = total + torch.nn.functional.cross_entropy(xx[src], tok[tgt].long(), reduction="sum")
        np.add.at(omega, src.numpy(), 1)
    (gamma * total).backward()
    return float(total.detach()), omega, xx.grad.numpy()


@pytest.mark.parametrize("t", [trees.spec_example(), trees.fig4_unit(), trees.tiny(),
                               trees.Tree([-1, 0, 0, 2, -1], [0, 2, 0, 1, 3]),
                               trees.Tree([-1, 0, 0], [3, 2, 2], [1, 1, 2])], ids=lambda t: t.name)
def test_loss_equals_per_branch_cross_entropy(t):
    V = 37
    pk, N, x, tok = _setup(t, V, seed=N_SEED)
    gamma = 0.75
    ref_loss, ref_omega, ref_grad = _torch_branch_ce(pk, x, tok, gamma)
    lr, om, dx = oracle.loss(pk, tok, V, np.arange(N), x, gamma=gamma)
    assert abs(lr.sum() - ref_loss) <= 1e-11 * max(1.0, abs(ref_loss))
    assert np.array_equal(om, ref_omega)
    assert np.allclose(dx, ref_grad, rtol=1e-11, atol=1e-13)
    # accounting: sum Omega = sum_l (L_l - 1)
    assert om.sum() == sum(max(len(p) - 1, 0) for p in oracle.paths(pk))


N_SEED = 17


def test_target_side_node_mask():
    t = trees.fig4_unit()
    V = 11
    pk, N, x, tok = _setup(t, V, seed=3)
    node_mask = np.array([1, 1, 0, 1, 1, 0, 1, 1, 1], np.uint8)
    sup = node_mask[pk["node"]]
    ref_loss, ref_omega, ref_grad = _torch_branch_ce(pk, x, tok, 1.0, sup=sup)
    lr, om, dx = oracle.loss(pk, tok, V, np.arange(N), x, node_loss_mask=node_mask)
    assert abs(lr.sum() - ref_loss) < 1e-11
    assert np.array_equal(om, ref_omega)
    assert np.allclose(dx, ref_grad, rtol=1e-11, atol=1e-13)


def test_uniform_logits_closed_form():
    t = trees.fig4_unit()
    V = 50
    pk = oracle.pack(t.parent, t.length)
    N = pk["n_tokens"]
    tok = np.arange(N, dtype=np.int32) % V
    x = np.zeros((N, V))
    gamma = 2.0
    lr, om, dx = oracle.loss(pk, tok, V, np.arange(N), x, gamma=gamma)
    assert np.allclose(lr, om * math.log(V), rtol=1e-14, atol=0)
    # dlogits = gamma (Omega / V - sum_k e_{y_k})
    exp = np.tile((gamma * om / V)[:, None], (1, V))
    for idx in oracle.paths(pk):
        for p in range(len(idx) - 1):
            exp[idx[p], tok[idx[p + 1]]] -= gamma
    assert np.allclose(dx, exp, atol=1e-14)
    # Fig. 4 tree: root token predicts u's token for all 5 trajectories; u predicts v1 (x3), v5 (x2)
    # packed order (DFS): r, u, v1, leaf1..3, v5, leaf4, leaf5
    assert om.tolist() == [5, 5, 3, 0, 0, 0, 2, 0, 0]


def test_boundary_mode_excludes_diverging_tokens():
    t = trees.spec_example()
    V = 13
    pk, N, x, tok = _setup(t, V, seed=4)
    lr0, om0, _ = oracle.loss(pk, tok, V, np.arange(N), x, boundary_mode=0)
    lr1, om1, dx1 = oracle.loss(pk, tok, V, np.arange(N), x, boundary_mode=1)
    # root's last token (index 4) diverges to leaf a (5) and leaf b (8)
    assert om0[4] == 2 and om1[4] == 0 and not dx1[4].any()
    om0[4] = 0
    assert np.array_equal(om0, om1)


def test_row_subset_matches_full():
    t = trees.gen_agentic(400, root_len=50, seed=1)
    V = 29
    pk, N, x, tok = _setup(t, V, seed=8)
    lr, om, dx = oracle.loss(pk, tok, V, np.arange(N), x)
    rows = np.array([0, 5, 77, N - 1, 200])
    lr2, om2, dx2 = oracle.loss(pk, tok, V, rows, x[rows])
    assert np.array_equal(lr2, lr[rows]) and np.array_equal(om2, om[rows]) and np.array_equal(dx2, dx[rows])


def test_finite_difference_on_logits():
    t = trees.spec_example()
    V = 7
    pk, N, x, tok = _setup(t, V, seed=9)
    _, _, dx = oracle.loss(pk, tok, V, np.arange(N), x, gamma=1.0)
    rng = np.random.default_rng(0)
    eps = 1e-6
    for _ in range(8):
        i, c = int(rng.integers(0, N)), int(rng.integers(0, V))
        xp, xm = x.clone(), x.clone()
        xp[i, c] += eps
        xm[i, c] -= eps
        fp = oracle.loss(pk, tok, V, np.arange(N), xp)[0].sum()
        fm = oracle.loss(pk, tok, V, np.arange(N), xm)[0].sum()
        assert abs((fp - fm) / (2 * eps) - dx[i, c]) < 1e-6
