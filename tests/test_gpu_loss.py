"""GPU parity for the Gradient-Restoration loss (tt_restore_loss) and the fp64 sum-of-squares
(tt_grad_sqnorm) against the oracle."""
import numpy as np
import pytest

import oracle
from workloads import trees, tensors
from _util import to64

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tt():
    import paper_2511_00413_b200 as P
    P.lib()
    return P


def _compare(tt, t, V, rows=None, gamma=1.0, node_mask=None, boundary_mode=0, inplace=False, seed=0):
    import torch
    pk = tt.tt_pack(t.parent, t.length, t.term)
    N = pk.n_tokens
    x = tensors.logits_tensor(N, V, seed=seed)
    tok = tensors.token_ids(N, V, seed=seed + 1)
    xd = x.cuda()
    tl = torch.empty(N, dtype=torch.float32, device="cuda")
    sums, dl, _, err = tt.tt_restore_loss(pk, xd, tok.cuda(), grad_scale=gamma, node_loss_mask=node_mask,
                                          boundary_mode=boundary_mode, dlogits=xd if inplace else None, tok_loss=tl)
    torch.cuda.synchronize()
    assert int(err.item()) == 0
    opk = oracle.pack(t.parent, t.length, t.term)
    rows = np.arange(N) if rows is None else np.asarray(rows)
    lr, om, dx = oracle.loss(opk, tok.numpy(), V, rows, x[torch.as_tensor(rows)], gamma=gamma,
                             node_loss_mask=node_mask, boundary_mode=boundary_mode)
    g = to64(dl.cpu()[torch.as_tensor(rows)])
    tol = 2.0 ** -8 * np.abs(dx) + 1e-5 * abs(gamma) * np.maximum(om, 1.0)[:, None]
    assert np.all(np.abs(g - dx) <= tol)
    tlr = to64(tl.cpu())[rows]
    assert np.allclose(tlr, lr, rtol=1e-5, atol=1e-4 * np.maximum(om, 1).max())
    if len(rows) == N:
        s = sums.cpu().numpy()
        assert abs(s[0] - lr.sum()) <= 1e-5 * max(1.0, abs(lr.sum()))
        assert s[1] == om.sum()
    return sums


@pytest.mark.parametrize("t", [trees.spec_example(), trees.fig4_unit(), trees.tiny(),
                               trees.gen_agentic(600, root_len=100, seed=3),
                               trees.Tree([-1, 0, 0, 2, -1, 4, 4], [0, 20, 0, 7, 15, 0, 3]),
                               trees.Tree([-1, 0, 0], [13, 7, 5], [1, 2, 1])], ids=lambda t: t.name)
def test_loss_small_vocab(tt, t):
    _compare(tt, t, V=1000, gamma=0.5)


def test_loss_vocab_not_multiple_of_8_rows_padded(tt):
    # ld must be a multiple of 8; vocab may be smaller than ld (padding ignored)
    import torch
    t = trees.spec_example()
    pk = tt.tt_pack(t.parent, t.length)
    N, V, ld = 12, 37, 40
    x = tensors.logits_tensor(N, ld, seed=5)
    tok = tensors.token_ids(N, V, seed=6)
    sums, dl, _, err = tt.tt_restore_loss(pk, x.cuda(), tok.cuda(), vocab=V)
    torch.cuda.synchronize()
    opk = oracle.pack(t.parent, t.length)
    lr, om, dx = oracle.loss(opk, tok.numpy(), V, np.arange(N), x[:, :V])
    assert abs(sums.cpu()[0].item() - lr.sum()) < 1e-4
    g = to64(dl.cpu()[:, :V])
    assert np.all(np.abs(g - dx) <= 2.0 ** -8 * np.abs(dx) + 1e-5 * np.maximum(om, 1)[:, None])


def test_loss_vocab_padded_to_16(tt):
    # V % 8 != 0 with 16-element-aligned rows (ld = 4112): the generic kernel (no 16-byte bulk copies
    # of a ragged row, no writes into the padding)
    import torch
    t = trees.gen_agentic(400, root_len=60, seed=8)
    pk = tt.tt_pack(t.parent, t.length)
    N, V, ld = pk.n_tokens, 4100, 4112
    x = tensors.logits_tensor(N, ld, seed=15)
    tok = tensors.token_ids(N, V, seed=16)
    xd = x.cuda()
    dl = torch.full_like(xd, 7.0)
    sums, dl, _, err = tt.tt_restore_loss(pk, xd, tok.cuda(), vocab=V, dlogits=dl)
    torch.cuda.synchronize()
    assert int(err.item()) == 0
    opk = oracle.pack(t.parent, t.length)
    lr, om, dx = oracle.loss(opk, tok.numpy(), V, np.arange(N), x[:, :V])
    assert abs(sums.cpu()[0].item() - lr.sum()) <= 1e-5 * max(1.0, abs(lr.sum()))
    g = to64(dl.cpu()[:, :V])
    assert np.all(np.abs(g - dx) <= 2.0 ** -8 * np.abs(dx) + 1e-5 * np.maximum(om, 1)[:, None])
    assert torch.all(dl[:, V:] == 7.0)  # padding untouched


def test_loss_node_mask_and_boundary_mode(tt):
    t = trees.fig4_unit()
    mask = np.array([1, 1, 0, 1, 1, 0, 1, 1, 1], np.uint8)
    _compare(tt, t, V=64, node_mask=mask)
    _compare(tt, trees.spec_example(), V=64, boundary_mode=1)


def test_loss_inplace_alias(tt):
    _compare(tt, trees.gen_agentic(300, root_len=60, seed=2), V=2048, gamma=2.0, inplace=True)


def test_loss_full_vocab_wide_sampled(tt):
    """Config 4 at full size (V = 151,936, 12,835 rows, in-place as in the bench); the oracle
    checks a sample of rows including the 4K-prefix's last token (64 continuations)."""
    t = trees.config_tree("wide")
    rows = [0, 1, 4094, 4095, 4096, 8000, 12834, 12000]
    _compare(tt, t, V=151936, rows=rows, inplace=True, seed=9)


def test_loss_bad_token_sets_error(tt):
    import torch
    t = trees.spec_example()
    pk = tt.tt_pack(t.parent, t.length)
    x = tensors.logits_tensor(12, 64, seed=1).cuda()
    tok = torch.zeros(12, dtype=torch.int32)
    tok[3] = 64  # out of range
    sums, dl, _, err = tt.tt_restore_loss(pk, x, tok.cuda())
    torch.cuda.synchronize()
    assert int(err.item()) == 1
    assert np.isnan(sums.cpu()[0].item())


def test_sqnorm(tt):
    import torch
    for n, dt in ((1, torch.float32), (1000003, torch.bfloat16), (77, torch.float32)):
        x = torch.randn(n, generator=torch.Generator().manual_seed(n)).to(dt)
        out = tt.tt_grad_sqnorm(x.cuda())
        torch.cuda.synchronize()
        ref = float((to64(x) ** 2).sum())
        # fp32 sums of 8 exact squares per vector, fp64 across vectors (include/tt.h)
        assert abs(out.item() - ref) <= 1e-6 * max(ref, 1.0)
        out2 = tt.tt_grad_sqnorm(x.cuda())
        torch.cuda.synchronize()
        assert out2.item() == out.item()  # deterministic


def test_sqnorm3_matches_single(tt):
    import torch
    xs = [torch.randn(n, generator=torch.Generator().manual_seed(n)).to(torch.bfloat16).cuda()
          for n in (4096 * 128, 333 * 128, 17)]
    out = tt.tt_grad_sqnorm3(*xs)
    singles = [tt.tt_grad_sqnorm(x) for x in xs]
    torch.cuda.synchronize()
    for k in range(3):
        assert out[k].item() == singles[k].item()


@pytest.mark.parametrize("V", [8, 64, 4104, 262144], ids=lambda v: f"V{v}")
def test_loss_kernel_paths(tt, V):
    """Every loss kernel path against the oracle: the 4-CTA cluster kernel (V % 8 == 0, slices in
    shared memory; V = 8 leaves three CTAs of each cluster with empty slices), and the L2 ring
    kernel when a slice no longer fits shared memory (V = 262,144)."""
    t = trees.gen_agentic(300, root_len=50, seed=4)
    _compare(tt, t, V=V, gamma=1.5, inplace=(V == 4104), seed=V % 97)


def test_loss_many_continuations(tt):
    """A node with 300 continuations (300-entry target lists in the cluster kernel's per-row
    metadata) with a target-side node mask, and repeated target token ids at the branch point."""
    import torch
    par = [-1] + [0] * 300 + [1, 1]
    ln = [40] + [2] * 300 + [3, 4]
    t = trees.Tree(par, ln)
    mask = np.ones(len(par), np.uint8)
    mask[5:40] = 0
    _compare(tt, t, V=2048, node_mask=mask, seed=3)
    # repeated target ids at the branch point: all continuations start with the same token
    pk = tt.tt_pack(t.parent, t.length)
    N, V = pk.n_tokens, 512
    x = tensors.logits_tensor(N, V, seed=8)
    tok = tensors.token_ids(N, V, seed=9)
    starts = pk.arrays()["node_start"].cpu().numpy()
    tok[torch.as_tensor(starts[1:301].astype(np.int64))] = 7
    sums, dl, _, err = tt.tt_restore_loss(pk, x.cuda(), tok.cuda())
    torch.cuda.synchronize()
    opk = oracle.pack(t.parent, t.length)
    lr, om, dx = oracle.loss(opk, tok.numpy(), V, np.arange(N), x)
    g = to64(dl.cpu())
    assert np.all(np.abs(g - dx) <= 2.0 ** -8 * np.abs(dx) + 1e-5 * np.maximum(om, 1.0)[:, None])
    assert abs(sums.cpu()[0].item() - lr.sum()) <= 1e-5 * max(1.0, abs(lr.sum()))


def test_loss_cluster_plus_tail_split(tt):
    """>= 8 rows per SM: the 4-CTA clusters take the head rows and loss_pipe_kernel, on the SMs the
    clusters leave idle (side stream forked from / joined into the caller's), the tail rows — every
    row, the sums, a target-side mask and boundary mode 1 against the oracle."""
    t = trees.gen_agentic(2400, root_len=200, seed=5)
    mask = (np.arange(len(t.parent)) % 5 != 2).astype(np.uint8)
    n0 = tt.tt_launch_count()
    _compare(tt, t, V=4096, gamma=0.75, node_mask=mask, boundary_mode=1, inplace=True, seed=21)
    n_split = tt.tt_launch_count() - n0
    _compare(tt, t, V=4096, gamma=1.0, seed=22)
    # V % 16 != 0: no split (clusters only)
    n0 = tt.tt_launch_count()
    _compare(tt, t, V=4104, gamma=1.0, seed=23)
    n_plain = tt.tt_launch_count() - n0
    assert n_split == n_plain + 1  # the tail-row kernel ran in the split case (same pack launches)


def test_loss_graph_capture_matches_eager(tt):
    """tt_restore_loss captured into a CUDA graph (the side-stream fork/join is captured with it)
    replays to the eager result bit for bit."""
    import torch
    t = trees.gen_agentic(2400, root_len=200, seed=5)
    pk = tt.tt_pack(t.parent, t.length)
    N, V = pk.n_tokens, 4096
    x = tensors.logits_tensor(N, V, seed=31).cuda()
    tok = tensors.token_ids(N, V, seed=32).cuda()
    dl0 = torch.empty_like(x)
    sums0, _, _, _ = tt.tt_restore_loss(pk, x, tok, dlogits=dl0)
    torch.cuda.synchronize()
    dl1 = torch.empty_like(x)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        tt.tt_restore_loss(pk, x, tok, dlogits=dl1)  # warm-up outside capture
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            sums1, _, _, _ = tt.tt_restore_loss(pk, x, tok, dlogits=dl1)
    dl1.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(dl0, dl1)
    assert torch.equal(sums0, sums1)


def test_loss_first_call_inside_capture(tt):
    """On a thread that has never called tt_restore_loss, the first call happening inside a CUDA-graph
    capture creates no stream / event (the split is skipped for it) and still replays correctly
    (against the eager, split result: equal up to bf16 rounding)."""
    import threading
    import torch
    t = trees.gen_agentic(2400, root_len=200, seed=7)
    pk = tt.tt_pack(t.parent, t.length)
    N, V = pk.n_tokens, 4096
    x = tensors.logits_tensor(N, V, seed=41).cuda()
    tok = tensors.token_ids(N, V, seed=42).cuda()
    dl0 = torch.empty_like(x)
    sums0, _, _, _ = tt.tt_restore_loss(pk, x, tok, dlogits=dl0)
    torch.cuda.synchronize()
    box = {}

    def work():
        try:
            torch.cuda.set_device(x.device)
            dl1 = torch.empty_like(x)
            sums1 = torch.empty(2, dtype=torch.float64, device=x.device)
            err = torch.zeros(1, dtype=torch.int32, device=x.device)
            s = torch.cuda.Stream()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                tt.tt_restore_loss(pk, x, tok, dlogits=dl1, sums=sums1, d_err=err)
            g.replay()
            torch.cuda.synchronize()
            box["r"] = (dl1, sums1)
        except Exception as e:  # surfaced in the main thread
            box["e"] = e

    th = threading.Thread(target=work)
    th.start()
    th.join()
    assert "e" not in box, box.get("e")
    dl1, sums1 = box["r"]
    # the captured call ran unsplit (all rows on the clusters) while the eager one gave the tail rows
    # to loss_pipe_kernel: same arithmetic up to fp32 rounding order, so equal to bf16 rounding
    a, b = dl0.float(), dl1.float()
    assert torch.all((a - b).abs() <= 2.0 ** -8 * a.abs() + 1e-6)
    assert torch.allclose(sums0, sums1, rtol=1e-6, atol=0)


@pytest.mark.parametrize("cfg", ["agentic8k", "wide"])
def test_loss_full_vocab_every_row(tt, cfg):
    """Qwen3 vocabulary (V = 151,936) at a BASELINE config's full size, in place as in the bench: the
    per-token loss of EVERY row (cluster-kernel rows and the tail rows the idle SMs take) against the
    oracle, and dlogits element-wise on 192 rows (96 spread over the whole range, 96 from the last
    30%, where the tail-row kernel works), plus the fp64 sums."""
    import torch
    t = trees.config_tree(cfg, 0 if cfg == "agentic8k" else None)
    V = 151936
    pk = tt.tt_pack(t.parent, t.length, t.term)
    N = pk.n_tokens
    x = tensors.logits_tensor(N, V, seed=19)
    tok = tensors.token_ids(N, V, seed=20)
    xd = x.cuda()
    tl = torch.empty(N, dtype=torch.float32, device="cuda")
    sums, dl, _, err = tt.tt_restore_loss(pk, xd, tok.cuda(), dlogits=xd, tok_loss=tl)
    torch.cuda.synchronize()
    assert int(err.item()) == 0
    opk = oracle.pack(t.parent, t.length, t.term)
    rng = np.random.default_rng(5)
    sample = np.unique(np.concatenate([np.linspace(0, N - 1, 96).astype(np.int64),
                                       rng.choice(np.arange(int(0.7 * N), N), 96, replace=False)]))
    tl_all = to64(tl.cpu())
    lsum = 0.0
    osum = 0.0
    for r0 in range(0, N, 1024):
        rows = np.arange(r0, min(N, r0 + 1024))
        lr, om, dx = oracle.loss(opk, tok.numpy(), V, rows, x[r0:rows[-1] + 1])
        assert np.allclose(tl_all[rows], lr, rtol=1e-5, atol=1e-4 * max(1.0, om.max())), r0
        lsum += lr.sum()
        osum += om.sum()
        pick = sample[(sample >= r0) & (sample <= rows[-1])]
        if len(pick):
            g = to64(dl[torch.as_tensor(pick)].cpu())
            ref = dx[pick - r0]
            tol = 2.0 ** -8 * np.abs(ref) + 1e-5 * np.maximum(om[pick - r0], 1.0)[:, None]
            assert np.all(np.abs(g - ref) <= tol), r0
    s = sums.cpu().numpy()
    assert abs(s[0] - lsum) <= 1e-5 * abs(lsum)
    assert s[1] == osum
