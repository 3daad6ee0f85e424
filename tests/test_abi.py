"""CPU-side checks of the C ABI (no GPU needed): libtt.so loads, exports every function tt.h
declares, and the host-only tt_pack_plan agrees with the oracle's accounting and error codes."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
from workloads import trees

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def tt():
    from paper_2511_00413_b200 import build
    build.build()
    import paper_2511_00413_b200 as P
    P.lib()
    return P


def _declared():
    src = open(os.path.join(ROOT, "include", "tt.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = set(re.findall(r"\b(tt_[a-z0-9_]+)\s*\(", src))
    return sorted(names)


def test_exports_every_declared_symbol(tt):
    names = _declared()
    assert len(names) >= 12
    so = ctypes.CDLL(tt.lib_path())
    for n in names:
        assert hasattr(so, n), n


def test_binding_names_match_abi(tt):
    for n in ("tt_pack_plan", "tt_pack", "tt_attn_fwd", "tt_attn_bwd", "tt_restore_loss", "tt_grad_sqnorm"):
        assert callable(getattr(tt, n))


@pytest.mark.parametrize("seed", range(25))
def test_pack_plan_matches_oracle_accounting(tt, seed):
    rng = np.random.default_rng(1000 + seed)
    t = trees.gen_random_forest(rng, max_nodes=30, max_len=40, with_term=(seed % 4 == 0))
    info = tt.tt_pack_plan(t.parent, t.length, t.term)
    pk = oracle.pack(t.parent, t.length, t.term)
    pos = pk["pos"].astype(np.int64)
    w = pk["w"].astype(np.int64)
    assert info["n_tokens"] == pk["n_tokens"]
    assert info["n_traj"] == pk["n_traj"]
    assert info["n_linear_tokens"] == int(w.sum())
    assert info["n_pairs"] == int((pos + 1).sum())
    assert info["n_linear_pairs"] == int((w * (pos + 1)).sum())
    assert info["n_blk"] == -(-pk["n_tokens"] // 128)


def test_pack_plan_configs(tt):
    t = trees.config_tree("agentic8k", 0)
    info = tt.tt_pack_plan(t.parent, t.length)
    # seed 0 -> A = 1.13e7, A_lin = 5.35e7, token ratio 8.32
    assert info["n_tokens"] == 8192
    assert abs(info["n_pairs"] / 1.13e7 - 1) < 0.01
    assert abs(info["n_linear_pairs"] / 5.35e7 - 1) < 0.01
    assert abs(info["n_linear_tokens"] / 8192 - 8.32) < 0.01


@pytest.mark.parametrize("bad,code", [
    (([-1, 2, 1], [1, 1, 1]), 2), (([0], [1]), 2), (([-1, 5], [1, 1]), 2),
    (([-1, 0], [0, 0]), 3), (([-1, 0], [1, -1]), 1),
])
def test_pack_plan_errors(tt, bad, code):
    with pytest.raises(tt.TTError) as ei:
        tt.tt_pack_plan(*bad)
    assert ei.value.code == code


def test_deep_chain_plan(tt):
    t = trees.chain(10000, seg=1)
    info = tt.tt_pack_plan(t.parent, t.length)
    assert info["n_tokens"] == 10000
    assert info["n_pairs"] == 10000 * 10001 // 2


def test_missing_library_fails_loudly(monkeypatch):
    """No fallback: with libtt.so absent every entry point raises instead of computing elsewhere."""
    from paper_2511_00413_b200 import binding
    monkeypatch.setattr(binding, "_SO", "/nonexistent/libtt.so")
    monkeypatch.setattr(binding, "_lib", None)
    with pytest.raises(ImportError):
        binding.lib()
    with pytest.raises(ImportError):
        binding.tt_pack_plan([-1, 0], [3, 2])


def test_release_build_has_no_dev_switches(tt):
    """The shipped libtt.so is a release build: tt_build_flags() reports no TT_DEV, and none of the
    development A/B environment variables (ablations that skip work, variant sweeps, CTA orders) is
    even referenced by the binary, so a stray variable on a bench box cannot change the timed work."""
    assert tt.lib().tt_build_flags() & 1 == 0
    blob = open(tt.lib_path(), "rb").read()
    for name in (b"TT_DEBUG_FWD", b"TT_DEBUG_BWD", b"TT_CTA_ORDER", b"TT_LOSS_VARIANT", b"TT_LOSS_NOCOMPUTE",
                 b"TT_LOSS_SPLIT", b"TT_LOSS_MAXCL", b"TT_LOSS_DEBUG"):
        assert name not in blob, name


@pytest.mark.parametrize("name,hq,hkv", [("agentic8k", 32, 32), ("agentic8k", 32, 8), ("deep32k", 32, 8),
                                         ("wide", 32, 8), ("batch64k", 32, 8), ("tiny", 4, 4)])
def test_bwd_kernel_dispatch_rule_host(tt, name, hq, hkv):
    """tt_attn_bwd_kernel is host logic (no CUDA call): on a tt_packed carrying the pack's schedule
    statistics it picks the persistent backward when the mean number of 64-row query tiles per (key
    block, kv head) item is below 80.  sched_sum_nq is recomputed here from the oracle's
    subtree ends (queries that see key block kb: [128 kb, max E over the block)); fp32 / d = 64 -> SIMT."""
    from paper_2511_00413_b200.binding import TTPacked, TT_BF16, TT_FP32
    t = trees.config_tree(name)
    opk = oracle.pack(t.parent, t.length)
    E, N = np.asarray(opk["E"]), int(opk["n_tokens"])
    nb = (N + 127) // 128
    nq = [(int(E[kb * 128:(kb + 1) * 128].max()) + 63) // 64 - 2 * kb for kb in range(nb)]
    c = TTPacked()
    c.n_tokens, c.n_blk, c.sched_sum_nq, c.sched_max_nq = N, nb, sum(nq), max(nq)
    kern = ctypes.c_int32(-1)
    L = tt.lib()
    assert L.tt_attn_bwd_kernel(ctypes.byref(c), hq, hkv, 128, TT_BF16, ctypes.byref(kern)) == 0
    assert kern.value == (1 if sum(nq) * (hq // hkv) / nb >= 80 else 0)
    assert L.tt_attn_bwd_kernel(ctypes.byref(c), hq, hkv, 64, TT_FP32, ctypes.byref(kern)) == 0
    assert kern.value == 2
    assert L.tt_attn_bwd_kernel(ctypes.byref(c), 32, 5, 128, TT_BF16, ctypes.byref(kern)) != 0  # hq % hkv != 0
