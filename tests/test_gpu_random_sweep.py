"""Randomised GPU parity sweep against the fp64 oracle: random forests (arbitrary node ids, several
roots, zero-length nodes, explicit trajectory counts term[] that end trajectories early or duplicate
them) with node lengths that straddle 128-token tile edges, random GQA shapes, both the tcgen05 bf16
path (d = 128) and the SIMT fp32 test mode (d = 64), and the restoration loss on small vocabularies
with random node masks — every output compared element by element (attention O / LSE max-abs,
gradients rel-L2, loss rows) at the north-star tolerances."""
import math
import os

import numpy as np
import pytest

import oracle
from workloads import trees, tensors
from _util import TOL_G_BF16, TOL_G_FP32, TOL_O_BF16, TOL_O_FP32, max_abs, rel_l2, to64

pytestmark = pytest.mark.gpu

HEADS = [(1, 1), (2, 1), (4, 2), (4, 1), (3, 3), (8, 2)]
# TT_SWEEP_SCALE=k multiplies the number of random cases (extended stress runs; default 1)
_K = max(1, int(os.environ.get("TT_SWEEP_SCALE", "1")))


@pytest.fixture(scope="module")
def tt():
    import paper_2511_00413_b200 as P
    P.lib()
    return P


def _forest(seed):
    rng = np.random.default_rng(7000 + seed)
    max_len = int(rng.choice([9, 60, 200, 300]))
    t = trees.gen_random_forest(rng, max_nodes=int(rng.integers(2, 14)), max_len=max_len,
                                with_term=bool(seed % 3 == 0))
    return t, rng


def _on_path(opk):
    c = np.zeros(opk["n_tokens"], np.int64)
    for idx in oracle.paths(opk):
        c[idx] += 1
    return c > 0


@pytest.mark.parametrize("seed", range(24 * _K))
@pytest.mark.parametrize("mode", ["bf16_d128", "fp32_d64"])
def test_random_attention(tt, seed, mode):
    import torch
    t, rng = _forest(seed)
    hq, hkv = HEADS[seed % len(HEADS)]
    dt, d = ("bf16", 128) if mode == "bf16_d128" else ("fp32", 64)
    pk = tt.tt_pack(t.parent, t.length, t.term)
    N = pk.n_tokens
    q, k, v = tensors.qkv_tensors(N, hq, hkv, d, dt, seed=seed)
    G = tensors.grad_tensor(N, hq, d, dt, seed=seed + 500)
    scale = 1.0 / math.sqrt(d)
    qd, kd, vd, Gd = (x.cuda() for x in (q, k, v, G))
    o, lse = tt.tt_attn_fwd(pk, qd, kd, vd, scale)
    dq, dk, dv = tt.tt_attn_bwd(pk, qd, kd, vd, o, lse, Gd, restore=True, softmax_scale=scale)
    torch.cuda.synchronize()
    opk = oracle.pack(t.parent, t.length, t.term)
    oo, olse = oracle.attn_fwd(opk, q, k, v, scale)
    odq, odk, odv = oracle.attn_bwd(opk, q, k, v, G, scale)
    m = _on_path(opk)  # tokens on no trajectory (term = 0 leaves) have no defined per-branch output
    tol_o, tol_g = (TOL_O_BF16, TOL_G_BF16) if dt == "bf16" else (TOL_O_FP32, TOL_G_FP32)
    assert max_abs(o.cpu()[m], oo[m]) <= tol_o
    assert max_abs(lse.cpu()[:, m], olse[:, m]) <= tol_o
    for a, b in ((dq, odq), (dk, odk), (dv, odv)):
        a, b = to64(a)[m], b[m]
        if np.abs(b).max() == 0:
            assert np.abs(a).max() <= 1e-5
        else:
            assert rel_l2(a, b) <= tol_g


@pytest.mark.parametrize("seed", range(16 * _K))
def test_random_loss(tt, seed):
    import torch
    t, rng = _forest(seed + 100)
    pk = tt.tt_pack(t.parent, t.length, t.term)
    N = pk.n_tokens
    V = int(rng.choice([8, 40, 1000, 4104]))
    gamma = float(rng.choice([1.0, 0.25]))
    mask = (rng.random(len(t.parent)) < 0.8).astype(np.uint8) if seed % 2 else None
    bmode = int(seed % 4 == 3)
    x = tensors.logits_tensor(N, V, seed=seed)
    tok = tensors.token_ids(N, V, seed=seed + 1)
    tl = torch.empty(N, device="cuda", dtype=torch.float32)
    sums, dl, tl, err = tt.tt_restore_loss(pk, x.cuda(), tok.cuda(), grad_scale=gamma, node_loss_mask=mask,
                                           boundary_mode=bmode, tok_loss=tl)
    torch.cuda.synchronize()
    opk = oracle.pack(t.parent, t.length, t.term)
    lr, om, odx = oracle.loss(opk, tok.numpy(), V, np.arange(N), x, gamma=gamma, node_loss_mask=mask,
                              boundary_mode=bmode)
    assert int(err.item()) == 0
    got = to64(tl)
    assert np.allclose(got, lr, rtol=1e-5, atol=1e-4 * np.maximum(om, 1).max())
    s = sums.cpu().numpy()
    assert abs(s[0] - lr.sum()) <= 1e-5 * max(1.0, abs(lr.sum()))
    assert s[1] == om.sum()
    d = to64(dl)
    assert np.all(np.abs(d - odx) <= 2.0 ** -8 * np.abs(odx) + 1e-5 * abs(gamma) * np.maximum(om, 1.0)[:, None])
