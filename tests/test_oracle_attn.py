"""Pins for the oracle's attention forward / backward (oracle.cpp `oracle_attn_fwd/bwd`).

Pinned against (none of these re-types the oracle's per-branch loop):
  * library special case: a single-node tree == torch SDPA(is_causal=True) in fp64, forward and
    autograd backward;
  * brute force: dense masked softmax attention in torch fp64 over the whole packed sequence
    with the parent-walk mask; its autograd with upstream gradient (trajectory count) * G equals
    the oracle's branch sum (PAPER Eqs. 20-21);
  * finite differences of L = sum_l sum_p <G, O_l[p]>;
  * closed forms: a single token gives O = v, LSE = s q.k, dV = G;
  * invariants: the bitwise branch-invariance of the forward;
  * negative controls: a plain causal mask over the packed sequence, and upstream G without
    the trajectory count ("restore off"), both fail.
"""
import math

import numpy as np
import pytest
import torch

import oracle
from workloads import trees



@pytest.fixture(autouse=True, scope="module")
def _fp64_default():
    # fp64 default dtype for this module's tensors only (restored afterwards, so it cannot leak into
    # other modules' tensors, e.g. fp32 GPU outputs)
    prev = torch.get_default_dtype()
    torch.set_default_dtype(torch.float64)
    yield
    torch.set_default_dtype(prev)


def _rand(N, hq, hkv, d, seed):
    g = torch.Generator().manual_seed(seed)
    q = torch.randn(N, hq, d, generator=g, dtype=torch.float64)
    k = torch.randn(N, hkv, d, generator=g, dtype=torch.float64)
    v = torch.randn(N, hkv, d, generator=g, dtype=torch.float64)
    G = torch.randn(N, hq, d, generator=g, dtype=torch.float64)
    return q, k, v, G


def _dense_attn(q, k, v, mask, scale):
    """Brute-force dense masked attention in torch fp64 (GQA by head repetition)."""
    N, hq, d = q.shape
    g = hq // k.shape[1]
    kk = k.repeat_interleave(g, dim=1)
    vv = v.repeat_interleave(g, dim=1)
    S = torch.einsum("ihc,jhc->hij", q, kk) * scale
    S = S.masked_fill(~mask[None], float("-inf"))
    lse = torch.logsumexp(S, dim=-1)
    P = torch.softmax(S, dim=-1)
    o = torch.einsum("hij,jhc->ihc", P, vv)
    return o, lse


def _counts(pk):
    c = np.zeros(pk["n_tokens"], np.int64)
    for idx in oracle.paths(pk):
        c[idx] += 1
    return torch.tensor(c, dtype=torch.float64)


@pytest.mark.parametrize("hq,hkv,d", [(1, 1, 8), (4, 2, 16), (3, 3, 5)])
def test_single_branch_equals_sdpa(hq, hkv, d):
    N = 23
    pk = oracle.pack([-1], [N])
    q, k, v, G = _rand(N, hq, hkv, d, seed=hq * 10 + d)
    scale = 1 / math.sqrt(d)
    o, lse = oracle.attn_fwd(pk, q, k, v, scale)
    g = hq // hkv
    qt = q.transpose(0, 1).clone().requires_grad_(True)
    kt = k.repeat_interleave(g, 1).transpose(0, 1).clone().requires_grad_(True)
    vt = v.repeat_interleave(g, 1).transpose(0, 1).clone().requires_grad_(True)
    ref = torch.nn.functional.scaled_dot_product_attention(qt, kt, vt, is_causal=True, scale=scale)
    assert np.allclose(o, ref.detach().transpose(0, 1).numpy(), rtol=1e-12, atol=1e-12)
    # backward: autograd of SDPA with upstream G
    ref.backward(G.transpose(0, 1))
    dq, dk, dv = oracle.attn_bwd(pk, q, k, v, G, scale)
    assert np.allclose(dq, qt.grad.transpose(0, 1).numpy(), rtol=1e-10, atol=1e-11)
    dk_ref = kt.grad.transpose(0, 1).reshape(N, hkv, g, d).sum(2)
    dv_ref = vt.grad.transpose(0, 1).reshape(N, hkv, g, d).sum(2)
    assert np.allclose(dk, dk_ref.numpy(), rtol=1e-10, atol=1e-11)
    assert np.allclose(dv, dv_ref.numpy(), rtol=1e-10, atol=1e-11)


def _cases():
    rng = np.random.default_rng(123)
    out = [trees.spec_example(), trees.fig4_unit(), trees.tiny(),
           trees.Tree([-1, 0, 0, 2, -1], [0, 2, 0, 1, 3], name="zero_len_multiroot"),
           trees.Tree([-1, 0], [2, 2], [1, 2], name="term")]
    for _ in range(8):
        out.append(trees.gen_random_forest(rng, max_nodes=9, max_len=5, with_term=bool(rng.random() < 0.3)))
    return out


@pytest.mark.parametrize("t", _cases(), ids=lambda t: t.name)
def test_tree_equals_dense_brute_force(t):
    pk = oracle.pack(t.parent, t.length, t.term)
    N = pk["n_tokens"]
    hq, hkv, d = 4, 2, 6
    q, k, v, G = _rand(N, hq, hkv, d, seed=N)
    scale = 0.37
    mask = torch.tensor(oracle.dense_mask(pk))
    o, lse = oracle.attn_fwd(pk, q, k, v, scale)       # also asserts bitwise branch invariance
    # rows on no trajectory (tokens of a node with no terminating trajectory below) are not
    # defined by the per-branch definition; with default term every token is on a path
    on_path = _counts(pk) > 0
    od, lsed = _dense_attn(q, k, v, mask, scale)
    assert np.allclose(o[on_path.numpy()], od[on_path].numpy(), rtol=1e-12, atol=1e-12)
    assert np.allclose(lse[:, on_path.numpy()], lsed[:, on_path].numpy(), rtol=1e-12, atol=1e-12)
    # backward: autograd of the dense forward with upstream (trajectory count) * G (App. B)
    qq, kk, vv = (x.clone().requires_grad_(True) for x in (q, k, v))
    od2, _ = _dense_attn(qq, kk, vv, mask, scale)
    cnt = _counts(pk)
    (od2 * (cnt[:, None, None] * G)).sum().backward()
    dq, dk, dv = oracle.attn_bwd(pk, q, k, v, G, scale)
    for a, b in ((dq, qq.grad), (dk, kk.grad), (dv, vv.grad)):
        assert np.allclose(a, b.numpy(), rtol=1e-10, atol=1e-11)
    # negative control: upstream G without restoration differs whenever a shared
    # prefix feeds >= 2 trajectories
    if (cnt > 1).any() and N > 1:
        qq.grad = kk.grad = vv.grad = None
        od3, _ = _dense_attn(qq, kk, vv, mask, scale)
        (od3 * G).sum().backward()
        assert not np.allclose(dv, vv.grad.numpy(), rtol=1e-6, atol=1e-8)


def test_negative_control_plain_causal_leaks():
    """A plain causal mask over the packed sequence changes sibling-branch outputs."""
    t = trees.spec_example()
    pk = oracle.pack(t.parent, t.length)
    q, k, v, _ = _rand(12, 2, 2, 4, seed=5)
    o, _ = oracle.attn_fwd(pk, q, k, v, 0.5)
    oc, _ = _dense_attn(q, k, v, torch.tril(torch.ones(12, 12, dtype=torch.bool)), 0.5)
    b0 = pk["node_start"][2]
    assert not np.allclose(o[b0:], oc[b0:].numpy(), atol=1e-6)
    assert np.allclose(o[:b0], oc[:b0].numpy(), atol=1e-12)   # prefix + first leaf unaffected


def test_single_token_closed_form():
    pk = oracle.pack([-1], [1])
    q, k, v, G = _rand(1, 1, 1, 7, seed=9)
    o, lse = oracle.attn_fwd(pk, q, k, v, 0.3)
    assert np.array_equal(o[0, 0], v[0, 0].numpy())
    assert abs(lse[0, 0] - 0.3 * float(q[0, 0] @ k[0, 0])) < 1e-14
    dq, dk, dv = oracle.attn_bwd(pk, q, k, v, G, 0.3)
    assert np.allclose(dv[0, 0], G[0, 0].numpy(), atol=1e-15)
    assert np.allclose(dq, 0, atol=1e-15) and np.allclose(dk, 0, atol=1e-15)


def test_zero_upstream_gives_zero_grads():
    t = trees.fig4_unit()
    pk = oracle.pack(t.parent, t.length)
    q, k, v, G = _rand(9, 2, 1, 4, seed=3)
    dq, dk, dv = oracle.attn_bwd(pk, q, k, v, torch.zeros_like(G), 0.5)
    assert not dq.any() and not dk.any() and not dv.any()


def test_finite_differences():
    """Central differences of L = sum_l sum_p <G[idx_l[p]], O_l[p]> (eps 1e-6, rel <= 1e-6)."""
    t = trees.Tree([-1, 0, 0, 1, 1], [3, 2, 2, 1, 2])
    pk = oracle.pack(t.parent, t.length)
    N = pk["n_tokens"]
    q, k, v, G = _rand(N, 2, 1, 4, seed=11)
    scale = 0.5
    paths = oracle.paths(pk)

    def L(q_, k_, v_):
        o, _ = oracle.attn_fwd(pk, q_, k_, v_, scale)
        return sum(float((G[idx].numpy() * o[idx]).sum()) for idx in paths)

    dq, dk, dv = oracle.attn_bwd(pk, q, k, v, G, scale)
    rng = np.random.default_rng(0)
    eps = 1e-6
    for name, X, grad in (("q", q, dq), ("k", k, dk), ("v", v, dv)):
        for _ in range(6):
            idx = tuple(int(rng.integers(0, s)) for s in X.shape)
            Xp, Xm = X.clone(), X.clone()
            Xp[idx] += eps
            Xm[idx] -= eps
            args_p = {"q": q, "k": k, "v": v}
            args_m = dict(args_p)
            args_p[name], args_m[name] = Xp, Xm
            fd = (L(**{a + "_": b for a, b in args_p.items()}) - L(**{a + "_": b for a, b in args_m.items()})) / (2 * eps)
            an = grad[idx]
            assert abs(fd - an) <= 1e-6 * max(1.0, abs(an)), (name, idx, fd, an)


def test_want_rows_subset_matches_full():
    t = trees.gen_agentic(600, root_len=100, seed=2)
    pk = oracle.pack(t.parent, t.length)
    N = pk["n_tokens"]
    q, k, v, G = _rand(N, 2, 1, 8, seed=2)
    o, lse = oracle.attn_fwd(pk, q, k, v, 0.3)
    dq, dk, dv = oracle.attn_bwd(pk, q, k, v, G, 0.3)
    rng = np.random.default_rng(1)
    want = np.zeros(N, np.uint8)
    want[rng.choice(N, 40, replace=False)] = 1
    wk = np.zeros(N, np.uint8)
    wk[rng.choice(N, 25, replace=False)] = 1
    o2, lse2 = oracle.attn_fwd(pk, q, k, v, 0.3, want=want, check_invariant=False)
    m = want.astype(bool)
    assert np.array_equal(o2[m], o[m]) and np.array_equal(lse2[:, m], lse[:, m])
    dq2, dk2, dv2 = oracle.attn_bwd(pk, q, k, v, G, 0.3, want_q=want, want_k=wk)
    mk = wk.astype(bool)
    assert np.array_equal(dq2[m], dq[m])
    assert np.array_equal(dk2[mk], dk[mk]) and np.array_equal(dv2[mk], dv[mk])


def test_want_subset_thread_count_and_single_filters():
    """The sampled backward splits work over rows / keys only: identical bits at any thread count,
    and with only one of want_q / want_k given (the other outputs stay 0)."""
    t = trees.gen_agentic(500, root_len=120, seed=6)
    pk = oracle.pack(t.parent, t.length)
    N = pk["n_tokens"]
    q, k, v, G = _rand(N, 4, 2, 8, seed=4)
    dq, dk, dv = oracle.attn_bwd(pk, q, k, v, G, 0.3)
    rng = np.random.default_rng(3)
    wq = np.zeros(N, np.uint8)
    wq[rng.choice(N, 30, replace=False)] = 1
    wk = np.zeros(N, np.uint8)
    wk[:5] = 1                      # root keys: every row of every branch contributes
    wk[rng.choice(N, 10, replace=False)] = 1
    mq, mk = wq.astype(bool), wk.astype(bool)
    for nt in (1, 3, 8):
        a = oracle.attn_bwd(pk, q, k, v, G, 0.3, want_q=wq, nthreads=nt)
        assert np.array_equal(a[0][mq], dq[mq]) and not a[1].any()
        b = oracle.attn_bwd(pk, q, k, v, G, 0.3, want_k=wk, nthreads=nt)
        assert np.array_equal(b[1][mk], dk[mk]) and np.array_equal(b[2][mk], dv[mk]) and not b[0].any()
