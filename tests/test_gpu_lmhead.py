"""GPU parity for NEXT-f3 (tt_lmhead_loss: LM head + Gradient-Restoration CE, vocabulary-chunked, the
[N, V] logits never materialised) against the fp64 oracle (oracle/lmhead.py: materialised logits,
per-branch cross entropy, dH = dX W, dW = dX^T H).  Ragged vocabulary chunks, a single chunk, target-side
node mask + boundary mode, and real-valued trajectory weights (NEXT-f4)."""
from types import SimpleNamespace

import numpy as np
import pytest

import oracle
from oracle import lmhead as ol
from workloads import trees
from _util import rel_l2, to64

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tt():
    import paper_2511_00413_b200 as P
    P.lib()
    return P


CASES = [
    # name, tree, D, V, vocab_chunk, options
    ("agentic700_chunks", trees.gen_agentic(700, root_len=150, seed=3), 256, 5003, 1024, {}),
    ("agentic700_onechunk", trees.gen_agentic(700, root_len=150, seed=3), 128, 3000, 1 << 20, {"gamma": 0.5}),
    ("wide_mask_boundary", trees.gen_wide(prefix=200, n_leaves=9), 64, 2048, 600, {"mask": True, "boundary_mode": 1}),
    ("agentic500_weights", trees.gen_agentic(500, root_len=100, seed=6), 128, 4096, 1000, {"weights": True}),
    # explicit trajectory counts: node 1's second child carries no trajectory, so under boundary mode 1
    # node 1's last token keeps its (single live) target while node 0's last token (two live) is excluded
    ("term_boundary", SimpleNamespace(parent=[-1, 0, 0, 1, 1, 2, 2], length=[90, 70, 40, 130, 33, 20, 61],
                                      term=[0, 0, 0, 1, 0, 2, 0]), 64, 1500, 512, {"boundary_mode": 1}),
]


@pytest.mark.parametrize("name,t,D,V,vc,opt", CASES, ids=[c[0] for c in CASES])
def test_lmhead_loss_matches_oracle(tt, name, t, D, V, vc, opt):
    import torch
    term = getattr(t, "term", None)
    pk = tt.tt_pack(t.parent, t.length, term)
    N = pk.n_tokens
    g = torch.Generator().manual_seed(11)
    H = torch.randn(N, D, generator=g).to(torch.bfloat16)
    W = (2.0 / D ** 0.5 * torch.randn(V, D, generator=g)).to(torch.bfloat16)
    tok = torch.randint(0, V, (N,), generator=g, dtype=torch.int32)
    gamma = opt.get("gamma", 1.0)
    mask = None
    if opt.get("mask"):
        mask = (np.arange(len(t.parent)) % 3 != 1).astype(np.uint8)
    alpha = None
    if opt.get("weights"):
        alpha = np.random.default_rng(3).normal(0.4, 1.0, pk.info["n_traj"]).astype(np.float32)
        tt.tt_pack_weights(pk, alpha)
    tl = torch.empty(N, device="cuda", dtype=torch.float32)
    sums, dh, dw, tl, err = tt.tt_lmhead_loss(pk, H.cuda(), W.cuda(), tok.cuda(), grad_scale=gamma, vocab_chunk=vc,
                                              node_loss_mask=mask, boundary_mode=opt.get("boundary_mode", 0),
                                              tok_loss=tl)
    torch.cuda.synchronize()
    opk = oracle.pack(t.parent, t.length, term)
    r = ol.lmhead_loss(opk, to64(H), to64(W), tok.numpy(), gamma=gamma, node_loss_mask=mask,
                       boundary_mode=opt.get("boundary_mode", 0),
                       traj_weight=None if alpha is None else alpha.astype(np.float64))
    assert int(err.item()) == 0
    lr = r["loss_rows"]
    got = to64(tl)
    badr = np.flatnonzero(~(np.abs(got - lr) <= 1e-4 * np.maximum(1.0, np.abs(lr))))
    assert len(badr) == 0, (len(badr), badr[:10].tolist(), got[badr[:5]].tolist(), lr[badr[:5]].tolist())
    s = sums.cpu().numpy()
    assert abs(s[0] - lr.sum()) <= 1e-5 * max(1.0, abs(lr.sum()))
    assert abs(s[1] - r["omega_rows"].sum()) <= 1e-5 * max(1.0, abs(r["omega_rows"].sum()))
    assert rel_l2(dh, r["dH"]) <= 1e-2, rel_l2(dh, r["dH"])
    assert rel_l2(dw, r["dW"]) <= 1e-2, rel_l2(dw, r["dW"])


def test_lmhead_bad_token_sets_error(tt):
    import torch
    t = trees.gen_agentic(300, root_len=64, seed=2)
    pk = tt.tt_pack(t.parent, t.length)
    N, D, V = pk.n_tokens, 64, 1000
    H = torch.randn(N, D).to(torch.bfloat16).cuda()
    W = torch.randn(V, D).to(torch.bfloat16).cuda()
    tok = torch.randint(0, V, (N,), dtype=torch.int32)
    tok[5] = V + 3   # an out-of-range target: its predicting row reports NaN and the error word is set
    tl = torch.empty(N, device="cuda", dtype=torch.float32)
    sums, dh, dw, tl, err = tt.tt_lmhead_loss(pk, H, W, tok.cuda(), vocab_chunk=256, tok_loss=tl)
    torch.cuda.synchronize()
    assert int(err.item()) == 1
    assert torch.isnan(tl[4]).item()
