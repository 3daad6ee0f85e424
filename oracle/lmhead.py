"""LM head + Gradient-Restoration loss oracle — TEST INFRASTRUCTURE ONLY
(see oracle/__init__.py).

Plain fp64 definition: logits X = H W^T (numpy matmul, a library primitive), then the oracle's
per-branch next-token cross entropy (oracle.loss: every trajectory linearised, ordinary CE per
branch, summed; P:549 / readings R6-R8, R17, R20) giving per-row loss, Omega and dX; the LM head's
gradients are dH = dX W and dW = dX^T H.  Nothing is chunked: the [N, V] logits are materialised
(only small V in tests).

Pinned by tests/test_oracle_lmhead.py: torch fp64 autograd of sum over branches of
F.cross_entropy(H_l W^T, targets_l, reduction='sum') (an independent formulation that never forms
the tree or the restoration weights), and central finite differences on H and W entries.
"""
from __future__ import annotations

import numpy as np

from . import loss as _loss


def lmhead_loss(pk, H, W, tok, gamma=1.0, node_loss_mask=None, boundary_mode=0, traj_weight=None):
    """Returns dict(loss_rows, omega_rows, dH, dW) in fp64."""
    H = np.asarray(H, dtype=np.float64)
    W = np.asarray(W, dtype=np.float64)
    N, V = H.shape[0], W.shape[0]
    X = H @ W.T
    lr, om, dx = _loss(pk, tok, V, np.arange(N), X, gamma=gamma, node_loss_mask=node_loss_mask,
                       boundary_mode=boundary_mode, traj_weight=traj_weight)
    return {"loss_rows": lr, "omega_rows": om, "dH": dx @ W, "dW": dx.T @ H}
