"""GPU parity for NEXT-f2 (position-embedding correction + Gradient Scaler through a full attention
block, Eqs. 17-23): tt_rope against the oracle's RoPE on restored positions, tt_restore_grad
bit-exact, and a whole block — QKV projections (cuBLAS via torch.matmul: plain library GEMMs),
tt_rope, tt_attn_fwd, O projection, then tt_restore_grad on the upstream gradient, tt_attn_bwd with
restore = 0 (the correction is transitive), inverse tt_rope and the projection backward — against the
oracle's per-branch block (oracle/block.py: every trajectory run as its own sequence with positions
0..L-1, gradients summed over branches)."""
import math

import numpy as np
import pytest

from oracle import block as ob
from workloads import trees
from _util import rel_l2, to64

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tt():
    import paper_2511_00413_b200 as P
    P.lib()
    return P


def _x(shape, seed, dtype, scale=1.0):
    import torch
    g = torch.Generator().manual_seed(seed)
    return (scale * torch.randn(*shape, generator=g)).to(dtype)


@pytest.mark.parametrize("dt,d,tol", [("bf16", 128, None), ("fp32", 128, 1e-5), ("bf16", 64, None), ("fp32", 64, 1e-5)])
@pytest.mark.parametrize("inverse", [False, True])
def test_rope_matches_oracle(tt, dt, d, tol, inverse):
    import torch
    dtype = torch.bfloat16 if dt == "bf16" else torch.float32
    t = trees.gen_agentic(3000, root_len=1200, seed=7)   # restored positions up to ~2.9K, several branches
    pk = tt.tt_pack(t.parent, t.length)
    N, H = pk.n_tokens, 3
    x = _x((N, H, d), 1, dtype)
    y = x.cuda().contiguous()
    tt.tt_rope(pk, y, base=1.0e6, inverse=inverse)
    pos = pk.arrays()["pos"].cpu().numpy()
    ref = ob.rope(torch.as_tensor(to64(x)), pos, base=1.0e6, inverse=inverse).numpy()
    err = np.abs(to64(y) - ref)
    bound = (2.0 ** -8) * np.abs(ref) + 1e-5 * float(np.abs(to64(x)).max()) if tol is None else tol * float(np.abs(to64(x)).max())
    assert np.all(err <= bound), float((err - bound).max())


def test_rope_large_positions_fp32(tt):
    import torch
    # one long node: positions up to 65535 (the batch64k scale); the fp64 angle reduction keeps fp32 accuracy
    t = trees.Tree(np.array([-1], np.int32), np.array([65536], np.int32), None)
    pk = tt.tt_pack(t.parent, t.length)
    x = _x((65536, 1, 128), 2, torch.float32)
    y = x.cuda().contiguous()
    tt.tt_rope(pk, y, base=1.0e6)
    ref = ob.rope(torch.as_tensor(to64(x)), np.arange(65536), base=1.0e6).numpy()
    assert np.abs(to64(y) - ref).max() <= 1e-5 * float(np.abs(to64(x)).max())


@pytest.mark.parametrize("dt", ["bf16", "fp32"])
def test_restore_grad_bit_exact(tt, dt):
    import torch
    dtype = torch.bfloat16 if dt == "bf16" else torch.float32
    t = trees.gen_agentic(900, root_len=200, seed=4)
    pk = tt.tt_pack(t.parent, t.length)
    N = pk.n_tokens
    g = _x((N, 2, 64), 3, dtype)
    gd = g.cuda().contiguous()
    tt.tt_restore_grad(pk, gd)
    w = pk.arrays()["w"].cpu().to(torch.float32)
    ref = (g.float() * w[:, None, None]).to(dtype)
    assert torch.equal(gd.cpu(), ref)
    # real-valued weights (NEXT-f4) replace the leaf counts
    alpha = np.random.default_rng(5).normal(0.2, 1.0, pk.info["n_traj"]).astype(np.float32)
    wr = tt.tt_pack_weights(pk, alpha)
    gd = g.cuda().contiguous()
    tt.tt_restore_grad(pk, gd)
    ref = (g.float() * wr[:N].cpu()[:, None, None]).to(dtype)
    assert torch.equal(gd.cpu(), ref)


def _gpu_block(tt, pk, X, Wq, Wk, Wv, Wo, G, hq, hkv, d, base):
    """The tree-training block on the GPU: every attention / RoPE / scaling step in libtt kernels,
    projections as plain cuBLAS GEMMs."""
    N = X.shape[0]
    q = (X @ Wq).view(N, hq, d).contiguous()
    k = (X @ Wk).view(N, hkv, d).contiguous()
    v = (X @ Wv).view(N, hkv, d).contiguous()
    tt.tt_rope(pk, q, base=base)                      # restored positions
    tt.tt_rope(pk, k, base=base)
    o, lse = tt.tt_attn_fwd(pk, q, k, v, 1 / math.sqrt(d))
    O = o.view(N, hq * d)
    Y = O @ Wo
    Gs = G.clone()
    tt.tt_restore_grad(pk, Gs)                        # Gradient Scaler before the backward
    dO = (Gs @ Wo.T).view(N, hq, d).contiguous()
    dWo = O.T @ Gs
    dq, dk, dv = tt.tt_attn_bwd(pk, q, k, v, o, lse, dO, restore=False, softmax_scale=1 / math.sqrt(d))
    tt.tt_rope(pk, dq, base=base, inverse=True)       # dX = R(-a) dY
    tt.tt_rope(pk, dk, base=base, inverse=True)
    dqf, dkf, dvf = dq.view(N, hq * d), dk.view(N, hkv * d), dv.view(N, hkv * d)
    return {"Y": Y, "dX": dqf @ Wq.T + dkf @ Wk.T + dvf @ Wv.T, "dWq": X.T @ dqf, "dWk": X.T @ dkf,
            "dWv": X.T @ dvf, "dWo": dWo}


BLOCK_CASES = [
    # name, tree, Dm, hq, hkv, d, dtype, tolerance (rel-L2 per tensor), trajectory weights
    ("agentic700_bf16", trees.gen_agentic(700, root_len=150, seed=3), 256, 4, 2, 128, "bf16", 3e-2, False),
    ("wide_bf16_weighted", trees.gen_wide(prefix=256, n_leaves=6), 128, 2, 1, 128, "bf16", 3e-2, True),
    ("agentic300_fp32", trees.gen_agentic(300, root_len=64, seed=4), 64, 2, 1, 64, "fp32", 1e-4, False),
]


@pytest.mark.parametrize("name,t,Dm,hq,hkv,d,dt,tol,weighted", BLOCK_CASES, ids=[c[0] for c in BLOCK_CASES])
def test_block_gradients_equal_branch_sum(tt, name, t, Dm, hq, hkv, d, dt, tol, weighted):
    import torch
    dtype = torch.bfloat16 if dt == "bf16" else torch.float32
    base = 1.0e6
    pk = tt.tt_pack(t.parent, t.length)
    N = pk.n_tokens
    X = _x((N, Dm), 10, dtype)
    Wq = _x((Dm, hq * d), 11, dtype, Dm ** -0.5)
    Wk = _x((Dm, hkv * d), 12, dtype, Dm ** -0.5)
    Wv = _x((Dm, hkv * d), 13, dtype, Dm ** -0.5)
    Wo = _x((hq * d, Dm), 14, dtype, (hq * d) ** -0.5)
    G = _x((N, Dm), 15, dtype)
    alpha = None
    if weighted:
        alpha = np.random.default_rng(16).uniform(0.25, 2.0, pk.info["n_traj"]).astype(np.float32)
        tt.tt_pack_weights(pk, alpha)
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False   # fp32 projections in fp32, not TF32
    try:
        got = _gpu_block(tt, pk, *(a.cuda() for a in (X, Wq, Wk, Wv, Wo, G)), hq, hkv, d, base)
        torch.cuda.synchronize()
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    ref = ob.block_branch_sum(t.parent, t.length, to64(X), to64(Wq), to64(Wk), to64(Wv), to64(Wo), to64(G),
                              hq, hkv, d, base=base, traj_weight=None if alpha is None else alpha.astype(np.float64))
    for key in ("Y", "dX", "dWq", "dWk", "dWv", "dWo"):
        e = rel_l2(got[key], ref[key])
        assert e <= tol, (key, e)

