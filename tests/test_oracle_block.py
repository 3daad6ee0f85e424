"""Pins of the NEXT-f2 block oracle (oracle/block.py) against things other than itself:
RoPE identities and its complex-number form, the torch SDPA library path on a one-node tree,
finite differences, the C++ per-branch attention oracle composed per token with restored
positions, and a negative control with packed indices as positions."""
import numpy as np
import pytest
import torch

import oracle
from oracle import block as ob
from workloads import trees


def _rand(shape, seed, scale=1.0):
    return np.random.default_rng(seed).standard_normal(shape) * scale


def test_rope_position_zero_is_identity():
    x = torch.as_tensor(_rand((5, 3, 8), 0))
    y = ob.rope(x, np.zeros(5, int))
    assert torch.equal(y, x)


def test_rope_preserves_pair_norms_and_inverts():
    x = torch.as_tensor(_rand((7, 2, 16), 1))
    pos = np.array([0, 1, 5, 100, 4096, 65535, 123456])
    y = ob.rope(x, pos, base=1.0e6)
    h = 8
    n0 = x[..., :h] ** 2 + x[..., h:] ** 2
    n1 = y[..., :h] ** 2 + y[..., h:] ** 2
    assert torch.allclose(n0, n1, rtol=1e-12, atol=1e-12)
    z = ob.rope(y, pos, base=1.0e6, inverse=True)
    assert torch.allclose(z, x, rtol=0, atol=1e-12)


def test_rope_equals_complex_multiplication():
    # independent formulation: z_j = x_j + i x_{j+d/2}, rotated by e^{i m base^(-2j/d)}
    d, base = 16, 10000.0
    x = _rand((6, 1, d), 2)
    pos = np.array([0, 3, 17, 250, 1000, 31999])
    z = x[..., : d // 2] + 1j * x[..., d // 2:]
    ang = pos[:, None, None] * base ** (-2.0 * np.arange(d // 2) / d)[None, None, :]
    zr = z * np.exp(1j * ang)
    ref = np.concatenate([zr.real, zr.imag], axis=-1)
    y = ob.rope(torch.as_tensor(x), pos, base=base).numpy()
    assert np.abs(y - ref).max() < 1e-12


def test_rope_scores_depend_only_on_relative_position():
    d = 32
    q = torch.as_tensor(_rand((1, 1, d), 3))
    k = torch.as_tensor(_rand((1, 1, d), 4))
    for m, n, sft in ((5, 2, 7), (100, 40, 1000), (9, 9, 12345)):
        a = (ob.rope(q, [m]) * ob.rope(k, [n])).sum()
        b = (ob.rope(q, [m + sft]) * ob.rope(k, [n + sft])).sum()
        assert abs(float(a - b)) < 1e-10 * max(1.0, abs(float(a)))


def _problem(tree, Dm, hq, hkv, d, seed):
    N = int(np.sum(tree.length))
    X = _rand((N, Dm), seed)
    Wq = _rand((Dm, hq * d), seed + 1, Dm ** -0.5)
    Wk = _rand((Dm, hkv * d), seed + 2, Dm ** -0.5)
    Wv = _rand((Dm, hkv * d), seed + 3, Dm ** -0.5)
    Wo = _rand((hq * d, Dm), seed + 4, (hq * d) ** -0.5)
    G = _rand((N, Dm), seed + 5)
    return X, Wq, Wk, Wv, Wo, G


def test_single_node_tree_equals_sdpa_autograd():
    Dm, hq, hkv, d = 12, 4, 2, 8
    t = trees.Tree(np.array([-1], np.int32), np.array([11], np.int32), None)
    X, Wq, Wk, Wv, Wo, G = _problem(t, Dm, hq, hkv, d, 10)
    r = ob.block_branch_sum(t.parent, t.length, X, Wq, Wk, Wv, Wo, G, hq, hkv, d, base=500.0)
    Xt = torch.as_tensor(X).requires_grad_()
    Ws = [torch.as_tensor(w).requires_grad_() for w in (Wq, Wk, Wv, Wo)]
    L = X.shape[0]
    pos = np.arange(L)
    q = ob.rope((Xt @ Ws[0]).view(L, hq, d), pos, 500.0).transpose(0, 1)
    k = ob.rope((Xt @ Ws[1]).view(L, hkv, d), pos, 500.0).transpose(0, 1)
    v = (Xt @ Ws[2]).view(L, hkv, d).transpose(0, 1)
    o = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=True)
    Y = o.transpose(0, 1).reshape(L, hq * d) @ Ws[3]
    (Y * torch.as_tensor(G)).sum().backward()
    assert np.abs(r["Y"] - Y.detach().numpy()).max() < 1e-12
    for key, ref in (("dX", Xt.grad), ("dWq", Ws[0].grad), ("dWk", Ws[1].grad), ("dWv", Ws[2].grad),
                     ("dWo", Ws[3].grad)):
        assert np.abs(r[key] - ref.numpy()).max() < 1e-11, key


def test_block_finite_differences():
    Dm, hq, hkv, d = 6, 2, 1, 4
    t = trees.Tree(np.array([-1, 0, 0, 1], np.int32), np.array([3, 2, 2, 1], np.int32), None)
    X, Wq, Wk, Wv, Wo, G = _problem(t, Dm, hq, hkv, d, 20)
    r = ob.block_branch_sum(t.parent, t.length, X, Wq, Wk, Wv, Wo, G, hq, hkv, d, base=100.0)

    def J(Wq_, Wk_, Wv_, Wo_, X_):
        rr = ob.block_branch_sum(t.parent, t.length, X_, Wq_, Wk_, Wv_, Wo_, G, hq, hkv, d, base=100.0)
        # J = sum over branches <G, Y_l> = sum_i w_i <G_i, Y_i> (every branch through i sees the same Y_i)
        return float((rr["w"][:, None] * G * rr["Y"]).sum())

    eps = 1e-6
    rng = np.random.default_rng(0)
    for name, arr, pos in (("dWq", Wq, 0), ("dWk", Wk, 1), ("dWv", Wv, 2), ("dWo", Wo, 3), ("dX", X, 4)):
        for _ in range(2):
            ij = tuple(rng.integers(0, s) for s in arr.shape)
            args = [Wq, Wk, Wv, Wo, X]
            up, dn = [a.copy() for a in args], [a.copy() for a in args]
            up[pos][ij] += eps
            dn[pos][ij] -= eps
            fd = (J(*up) - J(*dn)) / (2 * eps)
            an = r[name][ij]
            assert abs(fd - an) <= 1e-6 * max(1.0, abs(an)), (name, fd, an)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_tree_output_equals_per_token_composition_with_restored_positions(seed):
    Dm, hq, hkv, d, base = 16, 4, 2, 8, 1000.0
    rng = np.random.default_rng(300 + seed)
    t = trees.gen_random_forest(rng, max_nodes=8, max_len=6)
    X, Wq, Wk, Wv, Wo, G = _problem(t, Dm, hq, hkv, d, 30 + seed)
    r = ob.block_branch_sum(t.parent, t.length, X, Wq, Wk, Wv, Wo, G, hq, hkv, d, base=base)
    pk = oracle.pack(t.parent, t.length)
    N = pk["n_tokens"]

    def compose(pos):
        q = ob.rope(torch.as_tensor(X @ Wq).view(N, hq, d), pos, base).numpy()
        k = ob.rope(torch.as_tensor(X @ Wk).view(N, hkv, d), pos, base).numpy()
        v = (X @ Wv).reshape(N, hkv, d)
        o, _ = oracle.attn_fwd(pk, q, k, v, 1 / np.sqrt(d))
        return o.reshape(N, hq * d) @ Wo

    assert np.abs(compose(pk["pos"]) - r["Y"]).max() < 1e-10
    if N > int(t.length[0]) + 1 and len(oracle.paths(pk)) > 1:
        # negative control: packed indices as position ids break the equivalence
        assert np.abs(compose(np.arange(N)) - r["Y"]).max() > 1e-6


def test_trajectory_weights_scale_linearly():
    Dm, hq, hkv, d = 8, 2, 2, 4
    t = trees.Tree(np.array([-1, 0, 0], np.int32), np.array([4, 3, 2], np.int32), None)
    X, Wq, Wk, Wv, Wo, G = _problem(t, Dm, hq, hkv, d, 40)
    r1 = ob.block_branch_sum(t.parent, t.length, X, Wq, Wk, Wv, Wo, G, hq, hkv, d, traj_weight=[1.0, 0.0])
    r2 = ob.block_branch_sum(t.parent, t.length, X, Wq, Wk, Wv, Wo, G, hq, hkv, d, traj_weight=[0.0, 1.0])
    r3 = ob.block_branch_sum(t.parent, t.length, X, Wq, Wk, Wv, Wo, G, hq, hkv, d, traj_weight=[2.0, -0.5])
    for key in ("dX", "dWq", "dWk", "dWv", "dWo"):
        assert np.abs(2.0 * r1[key] - 0.5 * r2[key] - r3[key]).max() < 1e-12
