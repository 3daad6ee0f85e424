"""fp64 CPU oracle for the Tree Training hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference` leg may
import this package.  The product path (paper_2511_00413_b200/ and libtt.so) never imports, links
or executes anything under oracle/, and shares no code with it.

The arithmetic lives in oracle.cpp (plain C++17, fp64, -O2, no fast-math); this module only
marshals numpy / torch arrays through ctypes.  What each function computes, with the PAPER.md
passages it follows, is documented in oracle.cpp.

Parity status: every function is pinned by tests/test_oracle_*.py
against paper-printed values (Fig. 4gradient scales 5 and 3), SPEC worked examples,
closed forms, library special cases (torch SDPA / cross_entropy in fp64), brute force and finite
differences.  No function is "parity unpinned".
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_SO = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

ERRORS = {1: "invalid argument", 2: "not a forest", 3: "empty", 4: "too large",
          5: "forward branch-invariance assertion failed"}


class OracleError(RuntimeError):
    def __init__(self, code, what):
        super().__init__(f"oracle {what}: {ERRORS.get(code, code)}")
        self.code = code


def build(force: bool = False) -> str:
    """Compile liboracle.so with g++ (plain -O2, no fast-math)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        cmd = ["g++", "-std=c++17", "-O2", "-fPIC", "-shared", "-pthread", "-o", _SO, _SRC]
        subprocess.check_call(cmd)
    return _SO


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(_SO)
            i32p = C.POINTER(C.c_int32)
            i64p = C.POINTER(C.c_int64)
            u8p = C.POINTER(C.c_uint8)
            dp = C.POINTER(C.c_double)
            L.oracle_pack_sizes.argtypes = [i32p, i32p, i32p, C.c_int32, i64p, i64p, i64p]
            L.oracle_pack.argtypes = [i32p, i32p, i32p, C.c_int32] + [i32p] * 8 + [i64p, i32p]
            L.oracle_dense_mask.argtypes = [i32p, C.c_int32, C.c_int64, i32p, i32p, u8p]
            L.oracle_tiles.argtypes = [i32p, C.c_int32, C.c_int64, i32p, i32p, i32p, C.c_int32, u8p, i32p, i32p]
            L.oracle_attn_fwd.argtypes = [C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_double,
                                          dp, dp, dp, C.c_int64, i64p, i32p, u8p, C.c_int32, dp, dp, C.c_int32]
            L.oracle_attn_bwd.argtypes = [C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_double,
                                          dp, dp, dp, dp, C.c_int64, i64p, i32p, dp, u8p, u8p, dp, dp, dp, C.c_int32]
            L.oracle_loss.argtypes = [C.c_int64, C.c_int32, i32p, C.c_int64, i64p, i32p, dp, u8p, C.c_int32,
                                      C.c_double, C.c_int64, i64p, dp, dp, dp, dp, C.c_int32]
            _lib = L
    return _lib


def _ptr(a, ct):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(ct))


def _f64(x):
    """Exact upcast to fp64 numpy (torch bf16/fp32 or numpy)."""
    try:
        import torch
        if isinstance(x, torch.Tensor):
            return np.ascontiguousarray(x.detach().to("cpu", torch.float64).numpy())
    except ImportError:  # pragma: no cover
        pass
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


def _i32(x):
    return None if x is None else np.ascontiguousarray(np.asarray(x, dtype=np.int32))


def _u8(x):
    return None if x is None else np.ascontiguousarray(np.asarray(x, dtype=np.uint8))


def default_threads():
    return max(1, os.cpu_count() or 1)


def pack(parent, length, term=None) -> dict:
    """DFS pack of a forest (oracle.cpp `oracle_pack`).  Returns per-token pos/w/E/node, per-node
    start/sub_end/depth/leaves, and the trajectory CSR (path_ptr, path_idx)."""
    L = lib()
    parent = _i32(parent); length = _i32(length); term = _i32(term)
    n = int(parent.shape[0])
    N = C.c_int64(); T = C.c_int64(); P = C.c_int64()
    rc = L.oracle_pack_sizes(_ptr(parent, C.c_int32), _ptr(length, C.c_int32), _ptr(term, C.c_int32), n,
                             C.byref(N), C.byref(T), C.byref(P))
    if rc:
        raise OracleError(rc, "pack")
    N, T, P = N.value, T.value, P.value
    out = {k: np.zeros(N, np.int32) for k in ("pos", "w", "E", "node")}
    out.update({k: np.zeros(n, np.int32) for k in ("node_start", "node_sub_end", "node_depth", "node_leaves")})
    out["path_ptr"] = np.zeros(T + 1, np.int64)
    out["path_idx"] = np.zeros(max(P, 1), np.int32)
    rc = L.oracle_pack(_ptr(parent, C.c_int32), _ptr(length, C.c_int32), _ptr(term, C.c_int32), n,
                       *[_ptr(out[k], C.c_int32) for k in ("pos", "w", "E", "node", "node_start",
                                                          "node_sub_end", "node_depth", "node_leaves")],
                       _ptr(out["path_ptr"], C.c_int64), _ptr(out["path_idx"], C.c_int32))
    if rc:
        raise OracleError(rc, "pack")
    out["path_idx"] = out["path_idx"][:P]
    out["n_tokens"] = N
    out["n_traj"] = T
    out["parent"] = parent
    out["length"] = length
    return out


def _tw(pk, traj_weight):
    if traj_weight is None:
        return None
    a = np.ascontiguousarray(np.asarray(traj_weight, dtype=np.float64))
    if a.shape != (pk["n_traj"],):
        raise ValueError("traj_weight must have one entry per trajectory")
    return a


def paths(pk) -> list:
    """Trajectory index paths as a list of int arrays (ascending trajectory order)."""
    p = pk["path_ptr"]
    return [pk["path_idx"][p[t]:p[t + 1]] for t in range(len(p) - 1)]


def dense_mask(pk) -> np.ndarray:
    L = lib()
    N = pk["n_tokens"]
    m = np.zeros((N, N), np.uint8)
    rc = L.oracle_dense_mask(_ptr(pk["parent"], C.c_int32), len(pk["parent"]), N,
                             _ptr(pk["node"], C.c_int32), _ptr(pk["pos"], C.c_int32), _ptr(m, C.c_uint8))
    if rc:
        raise OracleError(rc, "dense_mask")
    return m.astype(bool)


def tiles(pk, B: int):
    """Brute-force tile classes [nb, nb] (0 empty, 1 partial, 2 full) and per-k-block min/max E."""
    L = lib()
    N = pk["n_tokens"]
    nb = (N + B - 1) // B
    cls = np.zeros((nb, nb), np.uint8)
    mn = np.zeros(nb, np.int32)
    mx = np.zeros(nb, np.int32)
    rc = L.oracle_tiles(_ptr(pk["parent"], C.c_int32), len(pk["parent"]), N, _ptr(pk["node"], C.c_int32),
                        _ptr(pk["pos"], C.c_int32), _ptr(pk["E"], C.c_int32), B, _ptr(cls, C.c_uint8),
                        _ptr(mn, C.c_int32), _ptr(mx, C.c_int32))
    if rc:
        raise OracleError(rc, "tiles")
    return cls, mn, mx


def attn_fwd(pk, q, k, v, scale, want=None, check_invariant=True, nthreads=None):
    """Tree attention forward by per-branch linearisation.  q [N,hq,d], k/v [N,hkv,d].
    Returns (o [N,hq,d], lse [hq,N]) in fp64; rows not in `want` are left at 0."""
    L = lib()
    q, k, v = _f64(q), _f64(k), _f64(v)
    N, hq, d = q.shape
    hkv = k.shape[1]
    o = np.zeros((N, hq, d))
    lse = np.zeros((hq, N))
    want = _u8(want)
    rc = L.oracle_attn_fwd(N, hq, hkv, d, float(scale), _ptr(q, C.c_double), _ptr(k, C.c_double),
                           _ptr(v, C.c_double), pk["n_traj"], _ptr(pk["path_ptr"], C.c_int64),
                           _ptr(pk["path_idx"], C.c_int32), _ptr(want, C.c_uint8), int(bool(check_invariant)),
                           _ptr(o, C.c_double), _ptr(lse, C.c_double), nthreads or default_threads())
    if rc:
        raise OracleError(rc, "attn_fwd")
    return o, lse


def attn_bwd(pk, q, k, v, g, scale, want_q=None, want_k=None, nthreads=None, traj_weight=None):
    """Tree attention backward = sum over branches of ordinary causal-attention gradients with
    per-token upstream gradient g [N,hq,d]; branch t weighted by traj_weight[t] when given (R20).
    Returns (dq, dk, dv) fp64."""
    L = lib()
    q, k, v, g = _f64(q), _f64(k), _f64(v), _f64(g)
    N, hq, d = q.shape
    hkv = k.shape[1]
    dq = np.zeros((N, hq, d))
    dk = np.zeros((N, hkv, d))
    dv = np.zeros((N, hkv, d))
    wq, wk = _u8(want_q), _u8(want_k)
    rc = L.oracle_attn_bwd(N, hq, hkv, d, float(scale), _ptr(q, C.c_double), _ptr(k, C.c_double),
                           _ptr(v, C.c_double), _ptr(g, C.c_double), pk["n_traj"],
                           _ptr(pk["path_ptr"], C.c_int64), _ptr(pk["path_idx"], C.c_int32),
                           _ptr(_tw(pk, traj_weight), C.c_double),
                           _ptr(wq, C.c_uint8), _ptr(wk, C.c_uint8), _ptr(dq, C.c_double),
                           _ptr(dk, C.c_double), _ptr(dv, C.c_double), nthreads or default_threads())
    if rc:
        raise OracleError(rc, "attn_bwd")
    return dq, dk, dv


def loss(pk, tok, vocab, row_ids, x_rows, gamma=1.0, node_loss_mask=None, boundary_mode=0, nthreads=None,
         traj_weight=None):
    """Per-branch next-token CE at the listed rows.  x_rows [n_rows, vocab] are the logits of
    row_ids.  node_loss_mask (nullable, per node) supervises a prediction iff the TARGET token's
    node is set (reading R17).  traj_weight (nullable, per trajectory) weights branch t's CE
    (R20).  Returns (loss_rows, omega_rows, dx_rows)."""
    L = lib()
    tok = _i32(tok)
    N = pk["n_tokens"]
    row_ids = np.ascontiguousarray(np.asarray(row_ids, dtype=np.int64))
    x = _f64(x_rows)
    n_rows = row_ids.shape[0]
    assert x.shape == (n_rows, vocab)
    sup = None
    if node_loss_mask is not None:
        sup = _u8(np.asarray(node_loss_mask, dtype=np.uint8)[pk["node"]])
    lr = np.zeros(n_rows); om = np.zeros(n_rows); dx = np.zeros((n_rows, vocab))
    rc = L.oracle_loss(N, vocab, _ptr(tok, C.c_int32), pk["n_traj"], _ptr(pk["path_ptr"], C.c_int64),
                       _ptr(pk["path_idx"], C.c_int32), _ptr(_tw(pk, traj_weight), C.c_double),
                       _ptr(sup, C.c_uint8), int(boundary_mode),
                       float(gamma), n_rows, _ptr(row_ids, C.c_int64), _ptr(x, C.c_double),
                       _ptr(lr, C.c_double), _ptr(om, C.c_double), _ptr(dx, C.c_double),
                       nthreads or default_threads())
    if rc:
        raise OracleError(rc, "loss")
    return lr, om, dx
