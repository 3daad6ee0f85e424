"""Full attention-block oracle — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Plain fp64 CPU PyTorch, written from the paper's definitions, slow on purpose:

  rope(x, pos, base, inverse)   RoPE "rotate-half" (reading R21): theta_j = base^(-2j/d), j < d/2,
                                 a = pos theta_j, (y_j, y_{j+d/2}) = (x_j cos a - x_{j+d/2} sin a,
                                 x_j sin a + x_{j+d/2} cos a); inverse rotates by -a.  Y = Rope(X, m)
                                 of P:509-515.
  block_branch_sum(...)         the PLAIN per-branch computation the method must reproduce
                                 (Eqs. 14-16 P:408-436 carried through the block, Eqs. 17-23
                                 P:440-517): for every trajectory l (root-to-leaf path, canonical
                                 order), gather its tokens X_l, run an ordinary causal attention block
                                 with positions 0..L_l-1
                                     Q = Rope(X_l Wq), K = Rope(X_l Wk), V = X_l Wv,
                                     O = softmax(scale Q K^T + causal) V  (GQA: kv head h // g),
                                     Y_l = O Wo,
                                 objective J = sum_l alpha_l <G[idx_l], Y_l> (alpha_l = 1 unless
                                 trajectory weights are given, reading R20), and gradients by fp64
                                 autograd of that per-branch program; dX is scatter-added over the
                                 branches, weight gradients summed.  Y per packed token is taken from
                                 the branches (asserted branch-invariant).

Pinned by tests/test_oracle_block.py: rope at position 0 is the identity, preserves every pair's
norm, depends only on relative position in q.k products, equals the complex-multiplication form
(x_j + i x_{j+d/2}) e^{i a}, and inverse o forward = id; the block on a one-node tree equals the
library path torch SDPA(is_causal) + autograd; central finite differences of J; the tree output
equals the per-token composition through the C++ attention oracle with restored positions; and a
negative control (packed indices as positions) breaks it.
"""
from __future__ import annotations

import numpy as np
import torch

from . import pack as _pack, paths as _paths


def rope(x, pos, base=1.0e6, inverse=False):
    """x [L, H, d] (torch fp64), pos [L] ints -> rotated copy (fp64)."""
    x = torch.as_tensor(x, dtype=torch.float64)
    L, H, d = x.shape
    half = d // 2
    j = torch.arange(half, dtype=torch.float64)
    theta = torch.pow(torch.tensor(float(base), dtype=torch.float64), -2.0 * j / d)        # [half]
    a = torch.as_tensor(np.asarray(pos), dtype=torch.float64)[:, None] * theta[None, :]    # [L, half]
    if inverse:
        a = -a
    c, s = torch.cos(a)[:, None, :], torch.sin(a)[:, None, :]
    x1, x2 = x[..., :half], x[..., half:]
    return torch.cat([x1 * c - x2 * s, x1 * s + x2 * c], dim=-1)


def _branch_forward(Xl, Wq, Wk, Wv, Wo, hq, hkv, d, base, scale):
    """One trajectory as an ordinary sequence: positions 0..L-1, causal attention (plain softmax)."""
    L = Xl.shape[0]
    g = hq // hkv
    pos = np.arange(L)
    q = rope((Xl @ Wq).view(L, hq, d), pos, base)
    k = rope((Xl @ Wk).view(L, hkv, d), pos, base)
    v = (Xl @ Wv).view(L, hkv, d)
    causal = torch.ones(L, L, dtype=torch.bool).tril()
    outs = []
    for h in range(hq):
        kh, vh = k[:, h // g, :], v[:, h // g, :]
        s = scale * (q[:, h, :] @ kh.T)
        s = s.masked_fill(~causal, float("-inf"))
        p = torch.softmax(s, dim=-1)
        outs.append(p @ vh)
    O = torch.stack(outs, dim=1).reshape(L, hq * d)
    return O @ Wo


def block_branch_sum(parent, length, X, Wq, Wk, Wv, Wo, G, hq, hkv, d, base=1.0e6, scale=None, term=None,
                     traj_weight=None):
    """Returns dict(Y [N, Dm], dX [N, Dm], dWq, dWk, dWv, dWo) in fp64 numpy (see module doc)."""
    scale = 1.0 / np.sqrt(d) if scale is None else float(scale)
    pk = _pack(parent, length, term)
    ps = _paths(pk)
    X = torch.as_tensor(np.asarray(X, dtype=np.float64))
    G = torch.as_tensor(np.asarray(G, dtype=np.float64))
    W = [torch.as_tensor(np.asarray(w, dtype=np.float64)).clone().requires_grad_() for w in (Wq, Wk, Wv, Wo)]
    N, Dm = X.shape
    Y = torch.full((N, Wo.shape[1]), float("nan"), dtype=torch.float64)
    dX = torch.zeros(N, Dm, dtype=torch.float64)
    alpha = np.ones(len(ps)) if traj_weight is None else np.asarray(traj_weight, dtype=np.float64)
    for l, idx in enumerate(ps):
        it = torch.as_tensor(np.asarray(idx, dtype=np.int64))
        Xl = X[it].clone().requires_grad_()
        Yl = _branch_forward(Xl, *W, hq, hkv, d, base, scale)
        J = float(alpha[l]) * (Yl * G[it]).sum()
        J.backward()
        dX.index_add_(0, it, Xl.grad)
        yl = Yl.detach()
        seen = ~torch.isnan(Y[it, 0])
        if bool(seen.any()):  # branch invariance of the forward, up to fp64 rounding order
            assert torch.allclose(Y[it][seen], yl[seen], rtol=1e-10, atol=1e-12)
        Y[it] = yl
    return {"Y": Y.numpy(), "dX": dX.numpy(), "dWq": W[0].grad.numpy(), "dWk": W[1].grad.numpy(),
            "dWv": W[2].grad.numpy(), "dWo": W[3].grad.numpy(), "pos": pk["pos"], "w": pk["w"]}
