"""GPU parity for real-valued leaf weights (NEXT-f4, tt_pack_weights): restoration in tt_attn_bwd and
tt_restore_loss with W_i = sum of alpha over the trajectories through token i, against the oracle's
alpha-weighted per-branch sums (reading R20), including traversal subsets of a capacity plan
("leaf weights present in THIS traversal")."""
import math

import numpy as np
import pytest

import oracle
from workloads import trees, tensors
from _util import TOL_G_BF16, TOL_G_FP32, rel_l2, to64

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tt():
    import paper_2511_00413_b200 as P
    P.lib()
    return P


def _alpha(n, seed, kind):
    rng = np.random.default_rng(seed)
    if kind == "advantage":
        return rng.normal(0.3, 1.0, n).astype(np.float32)  # any sign
    return rng.uniform(0.25, 2.0, n).astype(np.float32)


CASES = [
    ("agentic1500_bf16", trees.gen_agentic(1500, root_len=300, seed=5), 4, 2, 128, "bf16", "advantage"),
    ("wide_bf16", trees.gen_wide(prefix=512, n_leaves=7), 2, 1, 128, "bf16", "positive"),
    ("term_fp32", trees.Tree([-1, 0, 0], [130, 70, 5], [1, 2, 1]), 2, 1, 64, "fp32", "advantage"),
    ("agentic700_fp32", trees.gen_agentic(700, root_len=150, seed=3), 2, 2, 128, "fp32", "positive"),
]


@pytest.mark.parametrize("name,t,hq,hkv,d,dt,kind", CASES, ids=[c[0] for c in CASES])
def test_weighted_bwd(tt, name, t, hq, hkv, d, dt, kind):
    import torch
    pk = tt.tt_pack(t.parent, t.length, t.term)
    N = pk.n_tokens
    alpha = _alpha(pk.info["n_traj"], 1, kind)
    wr = tt.tt_pack_weights(pk, alpha)
    q, k, v = tensors.qkv_tensors(N, hq, hkv, d, dt, seed=2)
    G = tensors.grad_tensor(N, hq, d, dt, seed=3)
    qd, kd, vd, Gd = (x.cuda() for x in (q, k, v, G))
    scale = 1 / math.sqrt(d)
    o, lse = tt.tt_attn_fwd(pk, qd, kd, vd, scale)
    dq, dk, dv = tt.tt_attn_bwd(pk, qd, kd, vd, o, lse, Gd, restore=True, softmax_scale=scale)
    torch.cuda.synchronize()
    opk = oracle.pack(t.parent, t.length, t.term)
    # W on the device = fp64 subtree sums of alpha rounded once to fp32 (include/tt.h)
    W = np.zeros(N)
    for a, idx in zip(alpha.astype(np.float64), oracle.paths(opk)):
        W[idx] += a
    assert np.allclose(to64(wr[:N].cpu()), W, rtol=1e-6, atol=1e-6)
    assert np.all(wr[N:].cpu().numpy() == 0)
    odq, odk, odv = oracle.attn_bwd(opk, q, k, v, G, scale, traj_weight=alpha.astype(np.float64))
    tol = TOL_G_BF16 if dt == "bf16" else TOL_G_FP32
    for x, y in ((dq, odq), (dk, odk), (dv, odv)):
        assert rel_l2(x.cpu(), y) <= tol


def test_unit_weights_equal_integer_restore(tt):
    """alpha = 1 reproduces the integer tree-scale bit for bit (W = w exactly in fp32)."""
    import torch
    t = trees.gen_agentic(1200, root_len=200, seed=8)
    pk = tt.tt_pack(t.parent, t.length)
    N = pk.n_tokens
    q, k, v = tensors.qkv_tensors(N, 2, 1, 128, "bf16", seed=1)
    G = tensors.grad_tensor(N, 2, 128, "bf16", seed=2)
    qd, kd, vd, Gd = (x.cuda() for x in (q, k, v, G))
    o, lse = tt.tt_attn_fwd(pk, qd, kd, vd)
    ref = tt.tt_attn_bwd(pk, qd, kd, vd, o, lse, Gd, restore=True)
    tt.tt_pack_weights(pk, np.ones(pk.info["n_traj"], np.float32))
    got = tt.tt_attn_bwd(pk, qd, kd, vd, o, lse, Gd, restore=True)
    torch.cuda.synchronize()
    for a, b in zip(ref, got):
        assert torch.equal(a, b)


@pytest.mark.parametrize("kind", ["advantage", "positive"])
@pytest.mark.parametrize("size,V", [(600, 1000), (2400, 4096)], ids=["clusters", "clusters_plus_tail"])
def test_weighted_loss(tt, kind, size, V):
    """(2400, 4096): >= 8 rows per SM and V % 16 == 0, so the tail rows run in loss_pipe_kernel."""
    import torch
    t = trees.gen_agentic(size, root_len=100, seed=3)
    pk = tt.tt_pack(t.parent, t.length)
    N = pk.n_tokens
    alpha = _alpha(pk.info["n_traj"], 5, kind)
    tt.tt_pack_weights(pk, alpha)
    x = tensors.logits_tensor(N, V, seed=4)
    tok = tensors.token_ids(N, V, seed=5)
    tl = torch.empty(N, dtype=torch.float32, device="cuda")
    sums, dl, _, err = tt.tt_restore_loss(pk, x.cuda(), tok.cuda(), grad_scale=0.5, tok_loss=tl)
    torch.cuda.synchronize()
    assert int(err.item()) == 0
    opk = oracle.pack(t.parent, t.length)
    lr, om, dx = oracle.loss(opk, tok.numpy(), V, np.arange(N), x, gamma=0.5, traj_weight=alpha.astype(np.float64))
    g = to64(dl.cpu())
    # omega_k = W[target] rounded to fp32: relative 2^-24 on top of the bf16 output rounding
    tol = 2.0 ** -8 * np.abs(dx) + 1e-5 * 0.5 * np.maximum(np.abs(om), 1.0)[:, None]
    assert np.all(np.abs(g - dx) <= tol)
    scale_l = np.maximum(np.abs(lr), 1.0)
    assert np.all(np.abs(to64(tl.cpu()) - lr) <= 1e-4 * scale_l)
    s = sums.cpu().numpy()
    assert abs(s[0] - lr.sum()) <= 1e-5 * max(1.0, np.abs(lr).sum())
    assert abs(s[1] - om.sum()) <= 1e-5 * max(1.0, np.abs(om).sum())


def test_traversal_subset_weights(tt):
    """Each traversal of a capacity plan carries the weights of ITS trajectories only; summed over
    traversals the gradients equal the alpha-weighted branch sum over the whole tree."""
    import torch
    t = trees.gen_agentic(1800, root_len=300, seed=9)
    hq, hkv, d = 2, 1, 128
    opk = oracle.pack(t.parent, t.length)
    N = opk["n_tokens"]
    q, k, v = tensors.qkv_tensors(N, hq, hkv, d, "bf16", seed=6)
    G = tensors.grad_tensor(N, hq, d, "bf16", seed=7)
    scale = 1 / math.sqrt(d)
    alpha = _alpha(opk["n_traj"], 9, "advantage")
    a, info = tt.tt_plan_traversals(t.parent, t.length, 1000)
    assert info["n_traversals"] >= 2
    acc = [torch.zeros(N, h, d, dtype=torch.float64) for h in (hq, hkv, hkv)]
    for tr in range(info["n_traversals"]):
        par, ln, term, old = tt.tt_traversal_forest(t.parent, t.length, a, tr)
        idx = torch.as_tensor(np.flatnonzero(np.isin(opk["node"], old)))
        pk = tt.tt_pack(par, ln, term)
        tt.tt_pack_weights(pk, alpha[a == tr])  # canonical order is preserved by the induced forest
        qd, kd, vd, Gd = (x[idx].contiguous().cuda() for x in (q, k, v, G))
        o, lse = tt.tt_attn_fwd(pk, qd, kd, vd, scale)
        grads = tt.tt_attn_bwd(pk, qd, kd, vd, o, lse, Gd, restore=True, softmax_scale=scale)
        torch.cuda.synchronize()
        for s_, g_ in zip(acc, grads):
            s_.index_add_(0, idx, g_.cpu().double())
    ref = oracle.attn_bwd(opk, q, k, v, G, scale, traj_weight=alpha.astype(np.float64))
    for x, y in zip(acc, ref):
        assert rel_l2(x, y) <= TOL_G_BF16


def test_pack_weights_errors(tt):
    t = trees.spec_example()
    pk = tt.tt_pack(t.parent, t.length)
    with pytest.raises(ValueError):
        tt.tt_pack_weights(pk, np.ones(pk.info["n_traj"] + 1, np.float32))
    bad = np.ones(pk.info["n_traj"], np.float32)
    bad[0] = np.nan
    with pytest.raises(tt.TTError) as ei:
        tt.tt_pack_weights(pk, bad)
    assert ei.value.code == 1
    other = tt.tt_pack([-1, 0], [4, 4])
    other.parent, other.length = pk.parent, pk.length  # forest no longer matches the pack
    with pytest.raises(tt.TTError):
        tt.tt_pack_weights(other, np.ones(pk.info["n_traj"], np.float32)[:other.info["n_traj"]])
