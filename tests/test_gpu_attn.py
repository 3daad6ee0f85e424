"""GPU parity for tree-masked attention (tt_attn_fwd / tt_attn_bwd) against the fp64 oracle.

Every comparison consumes the SAME seeded inputs (workloads.tensors) rounded to the run dtype; the
oracle upcasts them exactly.  Tolerances: tests/_util.py (BASELINE.json north_star)."""
import math

import numpy as np
import pytest

import oracle
from workloads import trees, tensors
from _util import TOL_G_BF16, TOL_G_FP32, TOL_O_BF16, TOL_O_FP32, max_abs, rel_l2, to64

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tt():
    import paper_2511_00413_b200 as P
    P.lib()
    return P


def _run(tt, t, hq, hkv, d, dtype, seed=0, restore=True):
    import torch
    pk = tt.tt_pack(t.parent, t.length, t.term)
    N = pk.n_tokens
    q, k, v = tensors.qkv_tensors(N, hq, hkv, d, dtype, seed=seed)
    G = tensors.grad_tensor(N, hq, d, dtype, seed=seed + 100)
    qd, kd, vd, Gd = (x.cuda() for x in (q, k, v, G))
    scale = 1.0 / math.sqrt(d)
    o, lse = tt.tt_attn_fwd(pk, qd, kd, vd, scale)
    dq, dk, dv = tt.tt_attn_bwd(pk, qd, kd, vd, o, lse, Gd, restore=restore, softmax_scale=scale)
    torch.cuda.synchronize()
    return pk, (q, k, v, G, scale), (o.cpu(), lse.cpu(), dq.cpu(), dk.cpu(), dv.cpu())


def _oracle(t, q, k, v, G, scale):
    opk = oracle.pack(t.parent, t.length, t.term)
    o, lse = oracle.attn_fwd(opk, q, k, v, scale)
    dq, dk, dv = oracle.attn_bwd(opk, q, k, v, G, scale)
    return opk, o, lse, dq, dk, dv


def _on_path(opk):
    c = np.zeros(opk["n_tokens"], np.int64)
    for idx in oracle.paths(opk):
        c[idx] += 1
    return c > 0


FP32_CASES = [
    ("tiny", trees.tiny(), 1, 1, 64),
    ("spec", trees.spec_example(), 2, 1, 64),
    ("fig4", trees.fig4_unit(), 2, 2, 128),
    ("agentic700", trees.gen_agentic(700, root_len=150, seed=3), 4, 2, 64),
    ("wide_small", trees.gen_wide(prefix=300, n_leaves=6), 2, 1, 128),
    ("zero_multiroot", trees.Tree([-1, 0, 0, 2, -1, 4, 4], [0, 140, 0, 33, 150, 0, 9]), 2, 2, 64),
    ("term", trees.Tree([-1, 0, 0], [130, 70, 5], [1, 2, 1]), 2, 1, 64),
]


@pytest.mark.parametrize("name,t,hq,hkv,d", FP32_CASES, ids=[c[0] for c in FP32_CASES])
def test_fp32_test_mode(tt, name, t, hq, hkv, d):
    pk, (q, k, v, G, scale), (o, lse, dq, dk, dv) = _run(tt, t, hq, hkv, d, "fp32", seed=7)
    opk, oo, olse, odq, odk, odv = _oracle(t, q, k, v, G, scale)
    m = _on_path(opk)
    assert max_abs(o[m], oo[m]) <= TOL_O_FP32
    assert max_abs(lse[:, m], olse[:, m]) <= TOL_O_FP32
    for a, b in ((dq, odq), (dk, odk), (dv, odv)):
        assert rel_l2(a, b) <= TOL_G_FP32


BF16_CASES = [
    ("agentic1500_mha", trees.gen_agentic(1500, root_len=300, seed=5), 2, 2),
    ("agentic2000_gqa", trees.gen_agentic(2000, root_len=256, seed=1), 4, 1),
    ("wide_ragged", trees.gen_wide(prefix=512, n_leaves=7), 4, 2),
    ("chain_ragged", trees.chain(1, seg=999), 2, 1),
    ("single_token_nodes", trees.Tree([-1, 0, 0, 1, 1], [129, 1, 1, 130, 1]), 2, 2),
]


@pytest.mark.parametrize("name,t,hq,hkv", BF16_CASES, ids=[c[0] for c in BF16_CASES])
def test_bf16_tensor_core(tt, name, t, hq, hkv):
    tt.tt_launch_count_reset()
    pk, (q, k, v, G, scale), (o, lse, dq, dk, dv) = _run(tt, t, hq, hkv, 128, "bf16", seed=11)
    assert tt.tt_launch_count() >= 4
    opk, oo, olse, odq, odk, odv = _oracle(t, q, k, v, G, scale)
    assert max_abs(o, oo) <= TOL_O_BF16
    assert max_abs(lse, olse) <= TOL_O_BF16
    for a, b in ((dq, odq), (dk, odk), (dv, odv)):
        assert rel_l2(a, b) <= TOL_G_BF16
    # per-head relative errors too
    for h in range(hq):
        assert rel_l2(dq[:, h], odq[:, h]) <= TOL_G_BF16


def test_restore_off_negative_control(tt):
    """restore=0 with dO = G (no tree-scale) must miss the branch-sum gradient; restore=0
    with dO = w * G (already restored) must match it (R6)."""
    import torch
    t = trees.gen_agentic(900, root_len=200, seed=2)
    pk, (q, k, v, G, scale), (o, lse, dq0, dk0, dv0) = _run(tt, t, 2, 1, 128, "bf16", seed=3, restore=False)
    opk, oo, olse, odq, odk, odv = _oracle(t, q, k, v, G, scale)
    assert rel_l2(dv0, odv) > 0.1
    w = torch.tensor(opk["w"], dtype=torch.float32)
    Gw = (G.float() * w[:, None, None]).to(torch.bfloat16)
    qd, kd, vd = q.cuda(), k.cuda(), v.cuda()
    od, lsed = tt.tt_attn_fwd(pk, qd, kd, vd, scale)
    dq, dk, dv = tt.tt_attn_bwd(pk, qd, kd, vd, od, lsed, Gw.cuda(), restore=False, softmax_scale=scale)
    torch.cuda.synchronize()
    # Gw is rounded to bf16 after scaling, so compare against the oracle at the bf16 tolerance
    for a, b in ((dq, odq), (dk, odk), (dv, odv)):
        assert rel_l2(a.cpu(), b) <= TOL_G_BF16


def test_branch_invariance_on_gpu(tt):
    """The tree output at a shared-prefix token equals the output of the same kernels run on a
    linearised single branch, within bf16 tolerance."""
    import torch
    t = trees.gen_agentic(1200, root_len=400, seed=4)
    pk, (q, k, v, G, scale), (o, lse, *_ ) = _run(tt, t, 2, 2, 128, "bf16", seed=5)
    opk = oracle.pack(t.parent, t.length)
    idx = oracle.paths(opk)[-1]
    lin = tt.tt_pack([-1], [len(idx)])
    ii = torch.as_tensor(idx.astype(np.int64))
    ol, lsel = tt.tt_attn_fwd(lin, q[ii].contiguous().cuda(), k[ii].contiguous().cuda(), v[ii].contiguous().cuda(), scale)
    torch.cuda.synchronize()
    assert max_abs(ol.cpu(), o[ii]) <= 1e-2
    assert max_abs(lsel.cpu(), lse[:, ii]) <= 1e-3


@pytest.mark.parametrize("cfg,seed", [("agentic8k", 0), ("wide", None), ("deep32k", 1), ("batch64k", 0)])
def test_full_size_sampled_rows(tt, cfg, seed):
    """BASELINE configs at full size and the bench launch configuration; the oracle evaluates a
    sample of query rows (O, LSE, dQ) and of keys (dK, dV) one by one."""
    import torch
    t = trees.config_tree(cfg, seed)
    c = trees.CONFIGS[cfg]
    hq, hkv, d = c["hq"], c["hkv"], c["d"]
    pk, (q, k, v, G, scale), (o, lse, dq, dk, dv) = _run(tt, t, hq, hkv, d, "bf16", seed=21)
    opk = oracle.pack(t.parent, t.length)
    N = opk["n_tokens"]
    rng = np.random.default_rng(0)
    big = N > 20000
    want = np.zeros(N, np.uint8)
    want[rng.choice(N, 24 if big else 48, replace=False)] = 1
    want[[0, N - 1]] = 1
    # keys: leaf-level keys have short query ranges (cheap for the per-branch oracle)
    span = opk["E"] - np.arange(N)
    cand = np.flatnonzero(span <= (160 if big else 400))
    wk = np.zeros(N, np.uint8)
    wk[rng.choice(cand, min(8 if big else 24, len(cand)), replace=False)] = 1
    oo, olse = oracle.attn_fwd(opk, q, k, v, scale, want=want, check_invariant=False)
    m = want.astype(bool)
    assert max_abs(o[m], oo[m]) <= TOL_O_BF16
    assert max_abs(lse[:, m], olse[:, m]) <= TOL_O_BF16
    odq, odk, odv = oracle.attn_bwd(opk, q, k, v, G, scale, want_q=want, want_k=wk)
    mk = wk.astype(bool)
    assert rel_l2(dq[m], odq[m]) <= TOL_G_BF16
    assert rel_l2(dk[mk], odk[mk]) <= TOL_G_BF16
    assert rel_l2(dv[mk], odv[mk]) <= TOL_G_BF16


def test_unsupported_shapes_fail_loudly(tt):
    import torch
    pk = tt.tt_pack([-1], [64])
    q = torch.zeros(64, 2, 96, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(tt.TTError) as ei:
        tt.tt_attn_fwd(pk, q, q, q)
    assert ei.value.code == 5
    q = torch.zeros(64, 3, 128, dtype=torch.bfloat16, device="cuda")
    k = torch.zeros(64, 2, 128, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(tt.TTError):
        tt.tt_attn_fwd(pk, q, k, k)


def test_bwd_dk_dv_bitwise_deterministic(tt):
    """dK/dV accumulate in TMEM in a fixed order: repeated runs must be bitwise identical
    (guards the warpgroup hand-off of P^T / dS^T inside the backward kernel)."""
    import torch
    t = trees.gen_agentic(3000, root_len=600, seed=7)
    pk = tt.tt_pack(t.parent, t.length)
    N = pk.n_tokens
    q, k, v = (x.cuda() for x in tensors.qkv_tensors(N, 4, 2, 128, "bf16", seed=3))
    G = tensors.grad_tensor(N, 4, 128, "bf16", seed=4).cuda()
    o, lse = tt.tt_attn_fwd(pk, q, k, v)
    ref = [x.clone() for x in tt.tt_attn_bwd(pk, q, k, v, o, lse, G)]
    for _ in range(10):
        o2, lse2 = tt.tt_attn_fwd(pk, q, k, v)
        assert torch.equal(o2, o) and torch.equal(lse2, lse)
        d = tt.tt_attn_bwd(pk, q, k, v, o, lse, G)
        assert torch.equal(d[1], ref[1]) and torch.equal(d[2], ref[2])
        # dQ accumulates with fp32 reductions: order-dependent rounding only
        assert (d[0].float() - ref[0].float()).abs().max().item() <= 2e-2


EDGE_CASES = [
    # degenerate shapes on the tcgen05 path: one token, one partial block, exactly one block,
    # a forest of single-block roots with zero-length nodes, 1-token nodes straddling block edges
    ("one_token", trees.Tree([-1], [1]), 2, 1),
    ("one_partial_block", trees.Tree([-1, 0, 0], [40, 20, 17]), 2, 2),
    ("exactly_128", trees.Tree([-1, 0, 0], [64, 32, 32]), 2, 1),
    ("forest_zero_len", trees.Tree([-1, -1, 1, 1, -1, 4, 2], [127, 0, 129, 1, 255, 0, 2]), 4, 2),
    ("block_edge_nodes", trees.Tree([-1, 0, 1, 1, 0, 4], [127, 1, 128, 1, 1, 127]), 2, 2),
]


@pytest.mark.parametrize("name,t,hq,hkv", EDGE_CASES, ids=[c[0] for c in EDGE_CASES])
def test_bf16_edge_shapes(tt, name, t, hq, hkv):
    pk, (q, k, v, G, scale), (o, lse, dq, dk, dv) = _run(tt, t, hq, hkv, 128, "bf16", seed=13)
    opk, oo, olse, odq, odk, odv = _oracle(t, q, k, v, G, scale)
    m = _on_path(opk)
    assert max_abs(o[m], oo[m]) <= TOL_O_BF16
    assert max_abs(lse[:, m], olse[:, m]) <= TOL_O_BF16
    for a, b in ((dq, odq), (dk, odk), (dv, odv)):
        # a one-token tree has dQ = dK = 0 exactly (dS = P (dO.v - dO.O) with P = 1, O = v): there
        # the check is absolute (bf16 rounding of O leaves ~1e-8)
        assert rel_l2(a[m], b[m]) <= TOL_G_BF16 or (np.abs(to64(b[m])).max() == 0 and max_abs(a[m], b[m]) <= 1e-5)


def test_large_tree_sampled_rows(tt):
    """A ~100K-token tree (2K prefix, 400 leaves) — 790 query blocks, near the forward tile-list
    budget of one launch — checked on sampled rows / leaf keys."""
    import torch
    rng = np.random.default_rng(9)
    n_leaves = 400
    t = trees.Tree(np.array([-1] + [0] * n_leaves, np.int32),
                   np.array([2048] + list(rng.integers(150, 350, n_leaves)), np.int32))
    pk, (q, k, v, G, scale), (o, lse, dq, dk, dv) = _run(tt, t, 2, 1, 128, "bf16", seed=17)
    opk = oracle.pack(t.parent, t.length)
    N = opk["n_tokens"]
    assert N > 90000
    want = np.zeros(N, np.uint8)
    want[rng.choice(N, 40, replace=False)] = 1
    want[[0, N - 1]] = 1
    span = opk["E"] - np.arange(N)
    wk = np.zeros(N, np.uint8)
    wk[rng.choice(np.flatnonzero(span <= 300), 16, replace=False)] = 1
    oo, olse = oracle.attn_fwd(opk, q, k, v, scale, want=want, check_invariant=False)
    mq = want.astype(bool)
    assert max_abs(o[mq], oo[mq]) <= TOL_O_BF16
    assert max_abs(lse[:, mq], olse[:, mq]) <= TOL_O_BF16
    odq, odk, odv = oracle.attn_bwd(opk, q, k, v, G, scale, want_q=want, want_k=wk)
    mk = wk.astype(bool)
    assert rel_l2(dq[mq], odq[mq]) <= TOL_G_BF16
    assert rel_l2(dk[mk], odk[mk]) <= TOL_G_BF16
    assert rel_l2(dv[mk], odv[mk]) <= TOL_G_BF16


def test_too_many_blocks_fails_loudly(tt):
    """Beyond the forward kernel's tile-list budget the call returns TT_ERR_TOO_LARGE (no silent
    truncation, no fallback)."""
    import torch
    N = 512 * 1024
    pk = tt.tt_pack([-1], [N])
    q = torch.zeros(N, 1, 128, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(tt.TTError) as ei:
        tt.tt_attn_fwd(pk, q, q, q)
    assert ei.value.code == 4


@pytest.mark.parametrize("dt,d,hq,hkv", [("bf16", 128, 4, 2), ("bf16", 128, 2, 2), ("fp32", 64, 2, 1)])
def test_bwd_fused_sqnorm(tt, dt, d, hq, hkv):
    """Row a6 fused into tt_attn_bwd: ||dQ||^2, ||dK||^2, ||dV||^2 of the stored gradients, equal to a
    plain fp64 sum of squares and bitwise reproducible across runs."""
    import torch
    t = trees.gen_agentic(2500, root_len=500, seed=8)
    pk = tt.tt_pack(t.parent, t.length)
    N = pk.n_tokens
    q, k, v = (x.cuda() for x in tensors.qkv_tensors(N, hq, hkv, d, dt, seed=5))
    G = tensors.grad_tensor(N, hq, d, dt, seed=6).cuda()
    o, lse = tt.tt_attn_fwd(pk, q, k, v)
    outs = []
    for _ in range(3):
        nrm = torch.zeros(3, dtype=torch.float64, device="cuda")
        grads = tt.tt_attn_bwd(pk, q, k, v, o, lse, G, sqnorm=nrm)
        torch.cuda.synchronize()
        for i, x in enumerate(grads):
            ref = float((x.double() ** 2).sum())
            assert abs(float(nrm[i]) - ref) <= 1e-6 * ref, (i, float(nrm[i]), ref)
        outs.append(nrm.cpu())
    if dt == "bf16":  # dK/dV norms are bitwise reproducible (dK/dV are); dQ's follows dQ's rounding order
        assert torch.equal(outs[0][1:], outs[1][1:]) and torch.equal(outs[0][1:], outs[2][1:])


@pytest.mark.parametrize("cfg,seed", [("agentic8k", 0), ("wide", None), ("deep32k", 1)])
def test_full_size_tree_equals_linearised_kernels(tt, cfg, seed):
    """SURVEY §8(d) full-scale consistency (a property at any size, checked at the BASELINE sizes and
    bench launch configuration): the tree-packed fwd/bwd with restoration equals the same kernels run
    on every trajectory linearised as its own sequence, outputs gathered and gradients scatter-added
    back (Eqs. 14-16).  Not an oracle (it shares the kernels); the fp64 oracle covers sampled rows in
    test_full_size_sampled_rows."""
    import torch
    t = trees.config_tree(cfg, seed)
    c = trees.CONFIGS[cfg]
    hq, hkv, d = c["hq"], c["hkv"], c["d"]
    pk, (q, k, v, G, scale), (o, lse, dq, dk, dv) = _run(tt, t, hq, hkv, d, "bf16", seed=31)
    opk = oracle.pack(t.parent, t.length)
    paths = oracle.paths(opk)
    idx = torch.as_tensor(np.concatenate(paths).astype(np.int64))
    lin = tt.tt_pack([-1] * len(paths), [len(p) for p in paths])
    qd, kd, vd, Gd = (x.cuda() for x in (q, k, v, G))
    iq = idx.cuda()
    lq, lk, lv, lg = (x.index_select(0, iq).contiguous() for x in (qd, kd, vd, Gd))
    lo, llse = tt.tt_attn_fwd(lin, lq, lk, lv, scale)
    ldq, ldk, ldv = tt.tt_attn_bwd(lin, lq, lk, lv, lo, llse, lg, restore=False, softmax_scale=scale)
    torch.cuda.synchronize()
    # forward: every linearised occurrence of a token equals the tree output at that token
    assert max_abs(lo.cpu(), o[idx]) <= TOL_O_BF16
    # backward: scatter-add of the per-branch gradients equals the restored tree gradients
    for tree_g, lin_g, H in ((dq, ldq, hq), (dk, ldk, hkv), (dv, ldv, hkv)):
        acc = torch.zeros(o.shape[0], H, d, dtype=torch.float32, device="cuda")
        acc.index_add_(0, iq, lin_g.float())
        assert rel_l2(tree_g, acc.cpu()) <= TOL_G_BF16


def _root_key_case(tt, t, hq, hkv, seed, n_rows, key_blocks, full=False):
    """Tree whose first key blocks are seen by every query row (>= 256 query blocks of 128 rows):
    dK/dV of those root blocks accumulate over every q-tile x GQA head of the tree in one CTA, and
    dQ rows along the whole range receive ~N/128 key-block contributions.  Compared with the fp64
    oracle directly (rel-L2 per tensor and per head), not with the linearised kernels."""
    pk, (q, k, v, G, scale), (o, lse, dq, dk, dv) = _run(tt, t, hq, hkv, 128, "bf16", seed=seed)
    opk = oracle.pack(t.parent, t.length)
    N = opk["n_tokens"]
    assert N >= 256 * 128 and opk["E"][0] == N  # the root key block sees >= 256 query blocks
    rng = np.random.default_rng(seed)
    if full:
        wq = wk = None
        mq = mk = np.ones(N, bool)
    else:
        wq = np.zeros(N, np.uint8)
        wq[np.linspace(0, N - 1, n_rows).astype(np.int64)] = 1   # spread along the whole range
        wq[rng.choice(N, n_rows // 4, replace=False)] = 1
        wk = np.zeros(N, np.uint8)
        for kb in key_blocks:
            wk[kb * 128:min(N, kb * 128 + 128)] = 1
        mq, mk = wq.astype(bool), wk.astype(bool)
    oo, olse = oracle.attn_fwd(opk, q, k, v, scale, want=wq, check_invariant=False)
    assert max_abs(o[mq], oo[mq]) <= TOL_O_BF16
    assert max_abs(lse[:, mq], olse[:, mq]) <= TOL_O_BF16
    odq, odk, odv = oracle.attn_bwd(opk, q, k, v, G, scale, want_q=wq, want_k=wk)
    assert rel_l2(dq[mq], odq[mq]) <= TOL_G_BF16
    assert rel_l2(dk[mk], odk[mk]) <= TOL_G_BF16
    assert rel_l2(dv[mk], odv[mk]) <= TOL_G_BF16
    for h in range(hq):
        assert rel_l2(dq[mq][:, h], odq[mq][:, h]) <= TOL_G_BF16
    for h in range(hkv):
        assert rel_l2(dk[mk][:, h], odk[mk][:, h]) <= TOL_G_BF16
        assert rel_l2(dv[mk][:, h], odv[mk][:, h]) <= TOL_G_BF16
    # each root key block on its own (its 128 keys x heads), so a bad block cannot hide in the sum
    for kb in ([0, 1] if full else key_blocks):
        s = slice(kb * 128, kb * 128 + 128)
        assert rel_l2(dk[s], odk[s]) <= TOL_G_BF16 and rel_l2(dv[s], odv[s]) <= TOL_G_BF16


def test_root_keys_deep_prefix_vs_oracle(tt):
    """Deep shape (16K shared prefix, two 8.2K continuations, N = 32,768, GQA 4/1): the root key
    blocks walk all 256 query blocks x 4 heads (1,024 dK/dV accumulation steps of 128 rows) — the
    heaviest backward work of deep32k / batch64k, checked against the oracle."""
    t = trees.Tree([-1, 0, 0], [16384, 8192, 8192], name="deep_root")
    _root_key_case(tt, t, 4, 1, seed=41, n_rows=64, key_blocks=[0, 1, 63, 127, 128, 191, 255])


def test_root_keys_star_full_vs_oracle(tt):
    """Wide shape (256-token root + 255 leaves of 128, N = 32,896, GQA 8/2): the root key blocks see
    all 257 query blocks x 4 heads; every dQ / dK / dV element is compared with the oracle."""
    t = trees.star(256, [128] * 255)
    _root_key_case(tt, t, 8, 2, seed=43, n_rows=0, key_blocks=[], full=True)
