"""GPU check of capacity-constrained Tree Packing (NEXT-f1) end to end: the tree is split into
traversals by tt_plan_traversals, each traversal's induced sub-forest is packed and run through the
tensor-core attention forward/backward with Gradient Restoration, and the per-traversal gradients
scatter-added back equal the per-branch oracle over ALL trajectories ("multi-traversal
plan (C forces a split) vs run_baseline -> pass"); forward outputs agree on every token."""
import math

import numpy as np
import pytest

import oracle
from workloads import trees, tensors
from _util import TOL_G_BF16, TOL_O_BF16, max_abs, rel_l2

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("C", [900, 1100])
def test_multi_traversal_gradients_equal_branch_sum(C):
    import torch
    import paper_2511_00413_b200 as tt
    t = trees.gen_agentic(1800, root_len=300, seed=9)
    hq, hkv, d = 4, 2, 128
    opk = oracle.pack(t.parent, t.length)
    N = opk["n_tokens"]
    q, k, v = tensors.qkv_tensors(N, hq, hkv, d, "bf16", seed=4)
    G = tensors.grad_tensor(N, hq, d, "bf16", seed=5)
    scale = 1 / math.sqrt(d)
    a, info = tt.tt_plan_traversals(t.parent, t.length, C)
    assert info["n_traversals"] >= 2
    dq = torch.zeros(N, hq, d, dtype=torch.float64)
    dk = torch.zeros(N, hkv, d, dtype=torch.float64)
    dv = torch.zeros(N, hkv, d, dtype=torch.float64)
    o_all = torch.zeros(N, hq, d, dtype=torch.float64)
    for tr in range(info["n_traversals"]):
        par, ln, term, old = tt.tt_traversal_forest(t.parent, t.length, a, tr)
        # packed tokens of the induced forest = the original packed tokens of its nodes, in order
        keep = np.isin(opk["node"], old)
        idx = torch.as_tensor(np.flatnonzero(keep))
        pk = tt.tt_pack(par, ln, term)
        assert pk.n_tokens == len(idx) <= C
        qd, kd, vd, Gd = (x[idx].contiguous().cuda() for x in (q, k, v, G))
        o, lse = tt.tt_attn_fwd(pk, qd, kd, vd, scale)
        gq, gk, gv = tt.tt_attn_bwd(pk, qd, kd, vd, o, lse, Gd, restore=True, softmax_scale=scale)
        torch.cuda.synchronize()
        dq.index_add_(0, idx, gq.cpu().double())
        dk.index_add_(0, idx, gk.cpu().double())
        dv.index_add_(0, idx, gv.cpu().double())
        o_all[idx] = o.cpu().double()
    oo, _ = oracle.attn_fwd(opk, q, k, v, scale)
    odq, odk, odv = oracle.attn_bwd(opk, q, k, v, G, scale)
    assert max_abs(o_all, oo) <= TOL_O_BF16
    for x, y in ((dq, odq), (dk, odk), (dv, odv)):
        assert rel_l2(x, y) <= TOL_G_BF16
