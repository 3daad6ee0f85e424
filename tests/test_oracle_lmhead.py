"""Pins of the NEXT-f3 oracle (oracle/lmhead.py) against an independent formulation: torch fp64
autograd of the plain per-branch cross entropy of the LM head (no tree, no restoration weights),
and central finite differences."""
import numpy as np
import pytest
import torch

import oracle
from oracle import lmhead as ol
from workloads import trees


def _branch_ce(pk, H, W, tok):
    """sum over trajectories of F.cross_entropy(H_l W^T, next tokens, reduction='sum') + autograd."""
    Ht = torch.as_tensor(H).requires_grad_()
    Wt = torch.as_tensor(W).requires_grad_()
    total = 0.0
    for idx in oracle.paths(pk):
        idx = np.asarray(idx, dtype=np.int64)
        if len(idx) < 2:
            continue
        logits = Ht[idx[:-1]] @ Wt.T
        y = torch.as_tensor(np.asarray(tok)[idx[1:]].astype(np.int64))
        total = total + torch.nn.functional.cross_entropy(logits, y, reduction="sum")
    total.backward()
    return float(total), Ht.grad.numpy(), Wt.grad.numpy()


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_lmhead_oracle_equals_branch_autograd(seed):
    rng = np.random.default_rng(500 + seed)
    t = trees.gen_random_forest(rng, max_nodes=10, max_len=7)
    pk = oracle.pack(t.parent, t.length)
    N, D, V = pk["n_tokens"], 12, 37
    H = rng.standard_normal((N, D))
    W = rng.standard_normal((V, D)) * 0.5
    tok = rng.integers(0, V, N)
    r = ol.lmhead_loss(pk, H, W, tok)
    tot, dH, dW = _branch_ce(pk, H, W, tok)
    assert abs(r["loss_rows"].sum() - tot) <= 1e-10 * max(1.0, abs(tot))
    assert np.abs(r["dH"] - dH).max() < 1e-10
    assert np.abs(r["dW"] - dW).max() < 1e-10


def test_lmhead_oracle_finite_differences():
    rng = np.random.default_rng(7)
    t = trees.Tree(np.array([-1, 0, 0, 2], np.int32), np.array([3, 2, 2, 2], np.int32), None)
    pk = oracle.pack(t.parent, t.length)
    N, D, V = pk["n_tokens"], 5, 11
    H = rng.standard_normal((N, D))
    W = rng.standard_normal((V, D))
    tok = rng.integers(0, V, N)
    r = ol.lmhead_loss(pk, H, W, tok, gamma=1.0)
    eps = 1e-6
    for name, arr in (("dH", H), ("dW", W)):
        for _ in range(4):
            ij = tuple(rng.integers(0, s) for s in arr.shape)
            up, dn = arr.copy(), arr.copy()
            up[ij] += eps
            dn[ij] -= eps
            Hu, Wu = (up, W) if name == "dH" else (H, up)
            Hd, Wd = (dn, W) if name == "dH" else (H, dn)
            fd = (ol.lmhead_loss(pk, Hu, Wu, tok)["loss_rows"].sum() - ol.lmhead_loss(pk, Hd, Wd, tok)["loss_rows"].sum()) / (2 * eps)
            assert abs(fd - r[name][ij]) <= 1e-6 * max(1.0, abs(fd)), (name, fd, r[name][ij])
