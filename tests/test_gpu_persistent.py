"""GPU parity of the persistent attention kernels (cluster-launch-control work stealing, DESIGN.md §5.2,
§5.3) on forests with several work items per CTA: many small trees, so every CTA takes over several
(query-block pair, head) / (key block, kv head) items, many of them shorter than the kernels' claim /
prepare look-ahead (items of 1-3 query tiles), GQA and MHA.  Whole-tensor comparison against the fp64
oracle (Eqs. 1, 14-16, P:119-126 / P:408-436), plus bitwise reproducibility of dK / dV and of the fused
a6 scalars (an item's result must not depend on which CTA ran it or in which order)."""
import math

import numpy as np
import pytest

import oracle
from workloads import trees, tensors
from _util import TOL_G_BF16, TOL_O_BF16, max_abs, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tt():
    import paper_2511_00413_b200 as P
    P.lib()
    return P


def _forest(n_trees, seed, max_tokens=160):
    """n_trees small agentic trees side by side (one root each); lengths drawn so that most trees span
    one or two 128-token blocks."""
    rng = np.random.default_rng(seed)
    parent, length = [], []
    for i in range(n_trees):
        n = int(rng.integers(24, max_tokens))
        t = trees.gen_agentic(n, D=3, root_len=max(1, n // 3), seed=seed * 1000 + i)
        off = len(parent)
        parent.extend([-1 if p < 0 else p + off for p in t.parent])
        length.extend(int(x) for x in t.length)
    return trees.Tree(np.array(parent, np.int64), np.array(length, np.int64))


CASES = [
    ("gqa_8_2", 300, 8, 2, 11),
    ("mha_4_4", 260, 4, 4, 12),
]


@pytest.mark.parametrize("name,n_trees,hq,hkv,seed", CASES, ids=[c[0] for c in CASES])
def test_persistent_forest_matches_oracle(tt, name, n_trees, hq, hkv, seed):
    import torch
    t = _forest(n_trees, seed)
    pk = tt.tt_pack(t.parent, t.length)
    N, d = pk.n_tokens, 128
    nb = (N + 127) // 128
    assert nb * hkv > 2 * 148 and ((nb + 1) // 2) * hq > 2 * 148  # several items per CTA in both kernels
    assert tt.tt_attn_bwd_kernel(pk, hq, hkv) == "tree_attn_bwd_sm100"  # short items: the persistent kernel
    q, k, v = tensors.qkv_tensors(N, hq, hkv, d, "bf16", seed=seed)
    G = tensors.grad_tensor(N, hq, d, "bf16", seed=seed + 100)
    qd, kd, vd, Gd = (x.cuda() for x in (q, k, v, G))
    scale = 1.0 / math.sqrt(d)
    o, lse = tt.tt_attn_fwd(pk, qd, kd, vd, scale)
    nrm = torch.zeros(3, dtype=torch.float64, device="cuda")
    dq, dk, dv = tt.tt_attn_bwd(pk, qd, kd, vd, o, lse, Gd, restore=True, softmax_scale=scale, sqnorm=nrm)
    torch.cuda.synchronize()
    opk = oracle.pack(t.parent, t.length)
    oo, olse = oracle.attn_fwd(opk, q, k, v, scale)
    odq, odk, odv = oracle.attn_bwd(opk, q, k, v, G, scale)
    assert max_abs(o.cpu(), oo) <= TOL_O_BF16
    assert max_abs(lse.cpu(), olse) <= TOL_O_BF16
    for a, b in ((dq, odq), (dk, odk), (dv, odv)):
        assert rel_l2(a.cpu(), b) <= TOL_G_BF16
    # per kv head too: a mis-assigned item shows up as one head's block being wrong
    for hk in range(hkv):
        assert rel_l2(dk[:, hk].cpu(), odk[:, hk]) <= TOL_G_BF16
        assert rel_l2(dv[:, hk].cpu(), odv[:, hk]) <= TOL_G_BF16
    # fused a6 scalars equal the plain sums of squares of the stored gradients
    for i, x in enumerate((dq, dk, dv)):
        ref = float((x.double() ** 2).sum())
        assert abs(float(nrm[i]) - ref) <= 1e-6 * ref


def test_persistent_bitwise_reproducible(tt):
    """Items are taken over dynamically, so which CTA runs an item changes from run to run; dK, dV, O,
    LSE and the dK / dV norms must not."""
    import torch
    t = _forest(300, 21)
    pk = tt.tt_pack(t.parent, t.length)
    N, hq, hkv, d = pk.n_tokens, 8, 2, 128
    q, k, v = (x.cuda() for x in tensors.qkv_tensors(N, hq, hkv, d, "bf16", seed=3))
    G = tensors.grad_tensor(N, hq, d, "bf16", seed=4).cuda()
    runs = []
    for _ in range(3):
        o, lse = tt.tt_attn_fwd(pk, q, k, v)
        nrm = torch.zeros(3, dtype=torch.float64, device="cuda")
        dq, dk, dv = tt.tt_attn_bwd(pk, q, k, v, o, lse, G, restore=True, sqnorm=nrm)
        torch.cuda.synchronize()
        runs.append((o.clone(), lse.clone(), dk.clone(), dv.clone(), nrm.clone()))
    for r in runs[1:]:
        for a, b in zip(runs[0][:4], r[:4]):
            assert torch.equal(a, b)
        assert torch.equal(runs[0][4][1:], r[4][1:])


def test_bwd_kernel_dispatch(tt):
    """tt_attn_bwd_kernel reports the dispatch rule of DESIGN §5.3: the persistent kernel when the mean
    number of 64-row query tiles per (key block, kv head) item is below 80, the flat kernel above, SIMT for
    fp32 / d != 128; the rule is recomputed here from the tree (queries that see key block kb: [128 kb,
    maxE_kb))."""
    import torch
    for name, hq, hkv in (("agentic8k", 32, 32), ("deep32k", 32, 8), ("wide", 32, 8)):
        t = trees.config_tree(name)
        pk = tt.tt_pack(t.parent, t.length)
        opk = oracle.pack(t.parent, t.length)
        E, N = np.asarray(opk["E"]), opk["n_tokens"]
        nb = (N + 127) // 128
        nq = [(int(E[kb * 128:(kb + 1) * 128].max()) + 63) // 64 - 2 * kb for kb in range(nb)]
        per_item = sum(nq) * (hq // hkv) / nb
        want = "tree_attn_bwd_flat_sm100" if per_item >= 80 else "tree_attn_bwd_sm100"
        assert tt.tt_attn_bwd_kernel(pk, hq, hkv) == want, (name, per_item)
    t = trees.config_tree("agentic8k")
    pk = tt.tt_pack(t.parent, t.length)
    assert tt.tt_attn_bwd_kernel(pk, 32, 32) == "tree_attn_bwd_sm100"
    assert tt.tt_attn_bwd_kernel(pk, 4, 2, d=64, dtype=torch.float32) == "attn_bwd_simt"


def _random_big_forest(seed, n_parts):
    """n_parts random forests (zero-length nodes, several roots, explicit trajectory counts term[])
    concatenated: a forest with many short work items for the persistent kernels."""
    rng = np.random.default_rng(seed)
    parent, length, term = [], [], []
    for _ in range(n_parts):
        t = trees.gen_random_forest(rng, max_nodes=10, max_len=70, with_term=True)
        off = len(parent)
        parent.extend([-1 if p < 0 else int(p) + off for p in t.parent])
        length.extend(int(x) for x in t.length)
        term.extend(int(x) for x in t.term)
    return trees.Tree(np.array(parent, np.int64), np.array(length, np.int64), np.array(term, np.int64))


@pytest.mark.parametrize("seed,hq,hkv", [(31, 4, 4), (32, 8, 2), (33, 6, 3), (34, 4, 1)])
def test_persistent_random_forests(tt, seed, hq, hkv):
    """Random multi-item forests (ragged blocks, zero-length nodes, trajectories ending early or counted
    twice) through both persistent kernels, whole tensors against the oracle on the tokens some trajectory
    passes through (R12)."""
    import torch
    from _util import to64
    t = _random_big_forest(seed, 400)
    pk = tt.tt_pack(t.parent, t.length, t.term)
    N, d = pk.n_tokens, 128
    assert ((N + 127) // 128) * hkv > 148 and tt.tt_attn_bwd_kernel(pk, hq, hkv) == "tree_attn_bwd_sm100"
    q, k, v = tensors.qkv_tensors(N, hq, hkv, d, "bf16", seed=seed)
    G = tensors.grad_tensor(N, hq, d, "bf16", seed=seed + 100)
    qd, kd, vd, Gd = (x.cuda() for x in (q, k, v, G))
    scale = 1.0 / math.sqrt(d)
    o, lse = tt.tt_attn_fwd(pk, qd, kd, vd, scale)
    dq, dk, dv = tt.tt_attn_bwd(pk, qd, kd, vd, o, lse, Gd, restore=True, softmax_scale=scale)
    torch.cuda.synchronize()
    opk = oracle.pack(t.parent, t.length, t.term)
    oo, olse = oracle.attn_fwd(opk, q, k, v, scale)
    odq, odk, odv = oracle.attn_bwd(opk, q, k, v, G, scale)
    c = np.zeros(opk["n_tokens"], np.int64)
    for idx in oracle.paths(opk):
        c[idx] += 1
    m = c > 0
    assert max_abs(o.cpu()[m], oo[m]) <= TOL_O_BF16
    assert max_abs(lse.cpu()[:, m], olse[:, m]) <= TOL_O_BF16
    for a, b in ((dq, odq), (dk, odk), (dv, odv)):
        assert rel_l2(to64(a)[m], b[m]) <= TOL_G_BF16


def test_persistent_mixed_item_lengths(tt):
    """One 4K-token tree (items of up to ~256 query tiles) among 250 small trees: the dispatch
    still picks the persistent kernel (mean item length below the threshold), so long and short items
    share the persistent CTAs; whole tensors against the oracle and bitwise repeat."""
    import torch
    big = trees.gen_agentic(4096, D=5, p_open=0.3, root_len=1024, seed=77)
    small = _forest(250, 41)
    off = len(big.parent)
    parent = np.concatenate([np.asarray(big.parent, np.int64),
                             np.array([-1 if p < 0 else p + off for p in small.parent], np.int64)])
    length = np.concatenate([np.asarray(big.length, np.int64), np.asarray(small.length, np.int64)])
    t = trees.Tree(parent, length)
    pk = tt.tt_pack(t.parent, t.length)
    N, hq, hkv, d = pk.n_tokens, 8, 2, 128
    assert tt.tt_attn_bwd_kernel(pk, hq, hkv) == "tree_attn_bwd_sm100"
    assert pk.c.sched_max_nq * (hq // hkv) >= 200  # some items are long
    q, k, v = tensors.qkv_tensors(N, hq, hkv, d, "bf16", seed=5)
    G = tensors.grad_tensor(N, hq, d, "bf16", seed=6)
    qd, kd, vd, Gd = (x.cuda() for x in (q, k, v, G))
    scale = 1.0 / math.sqrt(d)
    outs = []
    for _ in range(2):
        o, lse = tt.tt_attn_fwd(pk, qd, kd, vd, scale)
        dq, dk, dv = tt.tt_attn_bwd(pk, qd, kd, vd, o, lse, Gd, restore=True, softmax_scale=scale)
        torch.cuda.synchronize()
        outs.append((o.cpu(), lse.cpu(), dq.cpu(), dk.cpu(), dv.cpu()))
    for a, b in zip(outs[0], outs[1]):
        if a is not outs[0][2]:  # dQ follows the fp32 reduction order; everything else is bitwise
            assert torch.equal(a, b)
    opk = oracle.pack(t.parent, t.length)
    oo, olse = oracle.attn_fwd(opk, q, k, v, scale)
    odq, odk, odv = oracle.attn_bwd(opk, q, k, v, G, scale)
    o, lse, dq, dk, dv = outs[0]
    assert max_abs(o, oo) <= TOL_O_BF16
    assert max_abs(lse, olse) <= TOL_O_BF16
    for a, b in ((dq, odq), (dk, odk), (dv, odv)):
        assert rel_l2(a, b) <= TOL_G_BF16
