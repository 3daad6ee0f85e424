"""ctypes binding of libtt.so — argument marshalling only (every step runs in the CUDA kernels).

Names mirror include/tt.h.  Tensors are torch tensors on the current CUDA device; the current
torch stream is passed as the tt_stream_t unless `stream` is given.  Workspaces are allocated
with torch (caching allocator) and owned by the returned Python objects.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import threading
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(HERE, "libtt.so")
TT_BLOCK = 128
TT_BF16, TT_FP32 = 0, 1

STATUS = {0: "ok", 1: "invalid argument", 2: "not a forest", 3: "empty", 4: "too large", 5: "unsupported",
          6: "alignment", 7: "workspace too small", 8: "cuda error"}


class TTError(RuntimeError):
    def __init__(self, fn, code, detail):
        super().__init__(f"{fn}: {STATUS.get(code, code)} ({detail})")
        self.code = code
        self.fn = fn


class TTPackInfo(C.Structure):
    _fields_ = [("n_nodes", C.c_int32), ("n_roots", C.c_int32), ("n_traj", C.c_int32), ("n_blk", C.c_int32),
                ("n_succ", C.c_int32), ("reserved", C.c_int32), ("n_tokens", C.c_int64),
                ("n_linear_tokens", C.c_int64), ("n_pairs", C.c_int64), ("n_linear_pairs", C.c_int64),
                ("ws_bytes", C.c_size_t)]


_PTR_FIELDS = ["pos", "w", "E", "node", "node_start", "node_len", "node_sub_end", "node_depth", "node_leaves",
               "succ_ptr", "succ_tok", "kblk_minE", "kblk_maxE", "fwd_cnt", "fwd_list", "wr"]


class TTPlanInfo(C.Structure):
    _fields_ = [("n_traj", C.c_int32), ("n_traversals", C.c_int32), ("capacity", C.c_int64),
                ("linear_tokens", C.c_int64), ("tree_tokens", C.c_int64), ("planned_tokens", C.c_int64)]


class TTPacked(C.Structure):
    _fields_ = [(f, C.c_void_p) for f in _PTR_FIELDS] + [
        ("n_tokens", C.c_int64), ("n_nodes", C.c_int32), ("n_blk", C.c_int32), ("n_succ", C.c_int32),
        ("max_succ", C.c_int32), ("sched_sum_nq", C.c_int64), ("sched_max_nq", C.c_int32), ("wr_negative", C.c_int32)]


_lock = threading.Lock()
_lib = None


def lib_path() -> str:
    return _SO


def lib():
    """Load libtt.so (raises if it is missing: no fallback path exists)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(_SO):
                raise ImportError(f"libtt.so not built at {_SO}; run `python -m paper_2511_00413_b200.build`")
            L = C.CDLL(_SO)
            i32p, vp, sz, st = C.POINTER(C.c_int32), C.c_void_p, C.c_size_t, C.c_void_p
            L.tt_status_string.restype = C.c_char_p
            L.tt_status_string.argtypes = [C.c_int]
            L.tt_last_error.restype = C.c_char_p
            L.tt_last_error.argtypes = []
            L.tt_version.restype = C.c_int32
            L.tt_build_flags.restype = C.c_int32
            L.tt_build_flags.argtypes = []
            L.tt_pack_plan.argtypes = [i32p, i32p, i32p, C.c_int32, C.POINTER(TTPackInfo)]
            L.tt_pack.argtypes = [i32p, i32p, i32p, C.c_int32, vp, sz, C.POINTER(TTPacked), C.POINTER(TTPackInfo), st]
            L.tt_attn_fwd.argtypes = [C.POINTER(TTPacked), vp, vp, vp, C.c_int, C.c_int32, C.c_int32, C.c_int32,
                                      C.c_float, vp, vp, st]
            L.tt_attn_bwd_workspace.argtypes = [C.POINTER(TTPacked), C.c_int32, C.c_int32, C.c_int32, C.c_int,
                                                C.POINTER(C.c_size_t)]
            L.tt_attn_bwd_kernel.argtypes = [C.POINTER(TTPacked), C.c_int32, C.c_int32, C.c_int32, C.c_int,
                                             C.POINTER(C.c_int32)]
            L.tt_attn_bwd.argtypes = [C.POINTER(TTPacked), vp, vp, vp, vp, vp, vp, C.c_int32, C.c_int, C.c_int32,
                                      C.c_int32, C.c_int32, C.c_float, vp, vp, vp, vp, vp, sz, st]
            L.tt_restore_loss_workspace.restype = C.c_size_t
            L.tt_restore_loss_workspace.argtypes = [C.POINTER(TTPacked)]
            L.tt_restore_loss.argtypes = [C.POINTER(TTPacked), vp, C.c_int64, C.c_int32, vp, vp, C.c_int32, C.c_float,
                                          vp, vp, vp, vp, vp, sz, st]
            L.tt_grad_sqnorm_workspace.restype = C.c_size_t
            L.tt_grad_sqnorm_workspace.argtypes = [C.c_int64]
            L.tt_grad_sqnorm.argtypes = [vp, C.c_int64, C.c_int, vp, vp, sz, st]
            L.tt_grad_sqnorm3.argtypes = [vp, C.c_int64, vp, C.c_int64, vp, C.c_int64, C.c_int, vp, vp, sz, st]
            L.tt_plan_traversals.argtypes = [i32p, i32p, i32p, C.c_int32, C.c_int64, i32p, C.POINTER(TTPlanInfo)]
            L.tt_pack_weights.argtypes = [i32p, i32p, i32p, C.c_int32, C.POINTER(C.c_float), C.POINTER(TTPacked),
                                          vp, st]
            L.tt_traversal_forest.argtypes = [i32p, i32p, i32p, C.c_int32, i32p, C.c_int32, i32p, i32p, i32p, i32p, i32p]
            L.tt_lmhead_loss_workspace.argtypes = [C.POINTER(TTPacked), C.c_int32, C.c_int32, C.c_int32,
                                                   C.POINTER(C.c_size_t)]
            L.tt_lmhead_loss.argtypes = [C.POINTER(TTPacked), vp, vp, C.c_int32, C.c_int32, C.c_int32, vp, vp, C.c_int32,
                                         C.c_float, vp, vp, vp, vp, vp, vp, sz, st]
            L.tt_rope.argtypes = [C.POINTER(TTPacked), vp, C.c_int, C.c_int32, C.c_int32, C.c_double, C.c_int32, st]
            L.tt_restore_grad.argtypes = [C.POINTER(TTPacked), vp, C.c_int, C.c_int64, st]
            L.tt_gemm.argtypes = [C.c_int32, C.c_int32, C.c_int32, vp, C.c_int64, C.c_int32, vp, C.c_int64, C.c_int32,
                                  vp, C.c_int64, C.c_int, C.c_int32, st]
            L.tt_launch_count.restype = C.c_int64
            L.tt_launch_count.argtypes = []
            L.tt_launch_count_reset.argtypes = []
            L.tt_launch_count_reset.restype = None
            for fn in ("tt_pack_plan", "tt_pack", "tt_attn_fwd", "tt_attn_bwd_workspace", "tt_attn_bwd_kernel", "tt_attn_bwd",
                       "tt_restore_loss", "tt_grad_sqnorm", "tt_grad_sqnorm3", "tt_plan_traversals",
                       "tt_traversal_forest", "tt_rope", "tt_restore_grad", "tt_lmhead_loss_workspace",
                       "tt_lmhead_loss", "tt_gemm"):
                getattr(L, fn).restype = C.c_int
            _lib = L
    return _lib


def _check(fn, rc):
    if rc != 0:
        raise TTError(fn, rc, lib().tt_last_error().decode(errors="replace"))


def _host_i32(x):
    if x is None:
        return None, None
    try:
        import torch
        if isinstance(x, torch.Tensor):
            x = x.detach().cpu().numpy()
    except ImportError:  # pragma: no cover
        pass
    a = np.ascontiguousarray(np.asarray(x, dtype=np.int32))
    return a, a.ctypes.data_as(C.POINTER(C.c_int32))


def _stream(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


def _dt(t):
    import torch
    if t.dtype == torch.bfloat16:
        return TT_BF16
    if t.dtype == torch.float32:
        return TT_FP32
    raise TypeError(f"unsupported dtype {t.dtype}")


def _p(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _need(t, dtype, name, device=None, contiguous=False):
    """Checks a caller-supplied tensor's dtype (the C ABI takes typed pointers: a mismatched torch
    dtype would be silently reinterpreted), and optionally its device and contiguity."""
    if t is None:
        return
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if device is not None and t.device != device:
        raise ValueError(f"{name} must be on {device}, got {t.device}")
    if contiguous and not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def _ws_stream(stream):
    """Context for allocating temporaries: on the stream the kernels run on, so the caching allocator
    never hands a still-in-use workspace to another stream (explicit stream= callers)."""
    import contextlib
    import torch
    if stream is None or not hasattr(stream, "cuda_stream"):
        return contextlib.nullcontext()
    return torch.cuda.stream(stream)


def tt_launch_count() -> int:
    return int(lib().tt_launch_count())


def tt_launch_count_reset() -> None:
    lib().tt_launch_count_reset()


def tt_pack_plan(parent, length, term=None) -> dict:
    """Host-only validation + sizing (no CUDA calls).  Returns the tt_pack_info fields."""
    par, pp = _host_i32(parent)
    ln, lp = _host_i32(length)
    tm, tp = _host_i32(term)
    info = TTPackInfo()
    _check("tt_pack_plan", lib().tt_pack_plan(pp, lp, tp, int(par.shape[0]), C.byref(info)))
    return {f: getattr(info, f) for f, _ in TTPackInfo._fields_ if f != "reserved"}


class PackedTree:
    """Result of tt_pack: the device workspace and the tt_packed struct pointing into it."""

    def __init__(self, c: TTPacked, info: dict, ws, parent, length, term):
        self.c = c
        self.info = info
        self.ws = ws
        self.parent, self.length, self.term = parent, length, term
        self.wr = None

    @property
    def n_tokens(self) -> int:
        return int(self.c.n_tokens)

    @property
    def n_blk(self) -> int:
        return int(self.c.n_blk)

    def _view(self, field: str, count: int):
        import torch
        off = getattr(self.c, field) - self.ws.data_ptr()
        return self.ws[off:off + 4 * count].view(torch.int32)

    def arrays(self) -> dict:
        """Device int32 views of every pack output (no copies)."""
        N, n, nb = self.n_tokens, int(self.c.n_nodes), self.n_blk
        out = {f: self._view(f, N) for f in ("pos", "w", "E", "node")}
        out.update({f: self._view(f, n) for f in ("node_start", "node_len", "node_sub_end", "node_depth",
                                                  "node_leaves")})
        out["succ_ptr"] = self._view("succ_ptr", n + 1)
        out["succ_tok"] = self._view("succ_tok", int(self.c.n_succ)) if self.c.n_succ else None
        out["kblk_minE"] = self._view("kblk_minE", nb)
        out["kblk_maxE"] = self._view("kblk_maxE", nb)
        out["fwd_cnt"] = self._view("fwd_cnt", nb)
        out["fwd_list"] = self._view("fwd_list", nb * (nb + 1) // 2)
        return out


def tt_pack(parent, length, term=None, device=None, stream=None) -> PackedTree:
    import torch
    par, pp = _host_i32(parent)
    ln, lp = _host_i32(length)
    tm, tp = _host_i32(term)
    info = TTPackInfo()
    L = lib()
    _check("tt_pack_plan", L.tt_pack_plan(pp, lp, tp, int(par.shape[0]), C.byref(info)))
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    ws = torch.empty(int(info.ws_bytes) + 256, dtype=torch.uint8, device=dev)
    # 256-byte aligned view
    mis = (-ws.data_ptr()) % 256
    ws = ws[mis:mis + int(info.ws_bytes)]
    c = TTPacked()
    info2 = TTPackInfo()
    _check("tt_pack", L.tt_pack(pp, lp, tp, int(par.shape[0]), C.c_void_p(ws.data_ptr()), int(info.ws_bytes),
                                C.byref(c), C.byref(info2), _stream(stream)))
    d = {f: getattr(info2, f) for f, _ in TTPackInfo._fields_ if f != "reserved"}
    d["max_succ"] = int(c.max_succ)
    return PackedTree(c, d, ws, par, ln, tm)


def tt_pack_weights(pk: PackedTree, traj_weight, stream=None):
    """Real-valued leaf weights (NEXT-f4): W_i = sum of traj_weight over the trajectories through
    token i (canonical trajectory order, include/tt.h).  Sets pk.c.wr; restoration in tt_attn_bwd
    and tt_restore_loss then uses W instead of the integer leaf count.  Returns the device W."""
    import numpy as np
    import torch
    a = np.ascontiguousarray(np.asarray(traj_weight, dtype=np.float32))
    if a.shape != (int(pk.info["n_traj"]),):
        raise ValueError(f"traj_weight must have n_traj = {pk.info['n_traj']} entries, got {a.shape}")
    par, pp = _host_i32(pk.parent)
    ln, lp = _host_i32(pk.length)
    tm, tp = _host_i32(pk.term)
    wr = torch.empty(pk.n_blk * 128, dtype=torch.float32, device=pk.ws.device)
    _check("tt_pack_weights", lib().tt_pack_weights(pp, lp, tp, int(par.shape[0]),
                                                    a.ctypes.data_as(C.POINTER(C.c_float)), C.byref(pk.c),
                                                    C.c_void_p(wr.data_ptr()), _stream(stream)))
    pk.wr = wr  # keep alive while pk references it
    return wr


def _scale(softmax_scale, d):
    return float(1.0 / math.sqrt(d)) if softmax_scale is None else float(softmax_scale)


def tt_attn_fwd(pk: PackedTree, q, k, v, softmax_scale=None, out=None, lse=None, stream=None):
    import torch
    N, hq, d = q.shape
    hkv = k.shape[1]
    if out is None:
        out = torch.empty_like(q)
    if lse is None:
        lse = torch.empty(hq, N, dtype=torch.float32, device=q.device)
    for t in (q, k, v, out, lse):
        if not t.is_contiguous():
            raise ValueError("tensors must be contiguous")
    _need(lse, torch.float32, "lse")
    _need(out, q.dtype, "out")
    _check("tt_attn_fwd", lib().tt_attn_fwd(C.byref(pk.c), _p(q), _p(k), _p(v), _dt(q), hq, hkv, d,
                                            _scale(softmax_scale, d), _p(out), _p(lse), _stream(stream)))
    return out, lse


def tt_attn_bwd_workspace(pk: PackedTree, hq, hkv, d, dtype) -> int:
    import torch
    n = C.c_size_t()
    dt = TT_BF16 if dtype == torch.bfloat16 else TT_FP32
    _check("tt_attn_bwd_workspace", lib().tt_attn_bwd_workspace(C.byref(pk.c), hq, hkv, d, dt, C.byref(n)))
    return int(n.value)


BWD_KERNELS = ("tree_attn_bwd_sm100", "tree_attn_bwd_flat_sm100", "attn_bwd_simt")


def tt_attn_bwd_kernel(pk: PackedTree, hq, hkv, d=128, dtype=None) -> str:
    """Name of the backward kernel tt_attn_bwd launches for this forest and head layout (host only)."""
    import torch
    dt = TT_FP32 if dtype == torch.float32 else TT_BF16
    kern = C.c_int32()
    _check("tt_attn_bwd_kernel", lib().tt_attn_bwd_kernel(C.byref(pk.c), hq, hkv, d, dt, C.byref(kern)))
    return BWD_KERNELS[kern.value]


def tt_attn_bwd(pk: PackedTree, q, k, v, o, lse, dout, restore=True, softmax_scale=None, dq=None, dk=None, dv=None,
                ws=None, sqnorm=None, stream=None):
    """sqnorm: optional fp64 device tensor [3] receiving ||dQ||^2, ||dK||^2, ||dV||^2 (fused, row a6)."""
    import torch
    N, hq, d = q.shape
    hkv = k.shape[1]
    with _ws_stream(stream):
        dq = torch.empty_like(q) if dq is None else dq
        dk = torch.empty_like(k) if dk is None else dk
        dv = torch.empty_like(v) if dv is None else dv
        need = tt_attn_bwd_workspace(pk, hq, hkv, d, q.dtype)
        if ws is None or ws.numel() < need:
            ws = torch.empty(need, dtype=torch.uint8, device=q.device)
    for name, t in (("k", k), ("v", v), ("o", o), ("dout", dout), ("dq", dq), ("dk", dk), ("dv", dv)):
        _need(t, q.dtype, name, q.device, contiguous=True)
    _need(q, q.dtype, "q", q.device, contiguous=True)
    _need(lse, torch.float32, "lse", q.device, contiguous=True)
    if tuple(o.shape) != tuple(q.shape) or tuple(dout.shape) != tuple(q.shape) or tuple(dq.shape) != tuple(q.shape):
        raise ValueError("o, dout, dq must have q's shape [N, hq, d]")
    if tuple(v.shape) != tuple(k.shape) or tuple(dk.shape) != tuple(k.shape) or tuple(dv.shape) != tuple(k.shape):
        raise ValueError("v, dk, dv must have k's shape [N, hkv, d]")
    _need(sqnorm, torch.float64, "sqnorm", q.device)
    _check("tt_attn_bwd", lib().tt_attn_bwd(C.byref(pk.c), _p(q), _p(k), _p(v), _p(o), _p(lse), _p(dout),
                                            int(bool(restore)), _dt(q), hq, hkv, d, _scale(softmax_scale, d),
                                            _p(dq), _p(dk), _p(dv), _p(sqnorm), _p(ws), int(ws.numel()),
                                            _stream(stream)))
    return dq, dk, dv


def tt_restore_loss(pk: PackedTree, logits, tok, grad_scale=1.0, node_loss_mask=None, boundary_mode=0,
                    dlogits=None, tok_loss=None, sums=None, d_err=None, ws=None, vocab=None, stream=None):
    """Returns (sums [2] fp64 device: (sum loss, sum Omega), dlogits, tok_loss, d_err).
    Pass dlogits=logits for the in-place (aliasing) form."""
    import torch
    if logits.dim() != 2 or logits.dtype != torch.bfloat16 or logits.stride(1) != 1:
        raise ValueError("logits must be a bf16 [N, V] tensor with unit column stride")
    N = logits.shape[0]
    ld = logits.stride(0)  # row stride in elements (a column-sliced view keeps its parent's stride)
    vocab = logits.shape[1] if vocab is None else int(vocab)
    if vocab > logits.shape[1]:
        raise ValueError(f"vocab {vocab} exceeds the logits width {logits.shape[1]}")
    dev = logits.device
    with _ws_stream(stream):
        dlogits = torch.empty_like(logits) if dlogits is None else dlogits
        sums = torch.zeros(2, dtype=torch.float64, device=dev) if sums is None else sums
        d_err = torch.zeros(1, dtype=torch.int32, device=dev) if d_err is None else d_err
        L = lib()
        need = int(L.tt_restore_loss_workspace(C.byref(pk.c)))
        if ws is None or ws.numel() < need:
            ws = torch.empty(need, dtype=torch.uint8, device=dev)
        if node_loss_mask is not None and not isinstance(node_loss_mask, torch.Tensor):
            node_loss_mask = torch.as_tensor(np.asarray(node_loss_mask, dtype=np.uint8), device=dev)
    if dlogits.dtype != torch.bfloat16 or tuple(dlogits.shape) != tuple(logits.shape) or dlogits.stride() != logits.stride():
        raise ValueError("dlogits must be bf16 with logits' shape and strides (or logits itself, in place)")
    if dlogits.device != dev:
        raise ValueError("dlogits must be on logits' device")
    if N != pk.n_tokens:
        raise ValueError(f"logits has {N} rows, the pack {pk.n_tokens} tokens")
    _need(tok, torch.int32, "tok", dev, contiguous=True)
    if tok.numel() < N:
        raise ValueError("tok must hold one token id per packed token")
    _need(node_loss_mask, torch.uint8, "node_loss_mask", dev, contiguous=True)
    _need(tok_loss, torch.float32, "tok_loss", dev, contiguous=True)
    _need(sums, torch.float64, "sums", dev, contiguous=True)
    _need(d_err, torch.int32, "d_err", dev)
    _check("tt_restore_loss", L.tt_restore_loss(C.byref(pk.c), _p(logits), int(ld), vocab, _p(tok),
                                                _p(node_loss_mask), int(boundary_mode), float(grad_scale),
                                                _p(dlogits), _p(tok_loss), _p(sums), _p(d_err), _p(ws),
                                                int(ws.numel()), _stream(stream)))
    return sums, dlogits, tok_loss, d_err


def tt_grad_sqnorm(x, out=None, ws=None, stream=None):
    import torch
    out = torch.zeros(1, dtype=torch.float64, device=x.device) if out is None else out
    L = lib()
    need = int(L.tt_grad_sqnorm_workspace(x.numel()))
    if ws is None or ws.numel() < need:
        ws = torch.empty(need, dtype=torch.uint8, device=x.device)
    _check("tt_grad_sqnorm", L.tt_grad_sqnorm(_p(x), int(x.numel()), _dt(x), _p(out), _p(ws), int(ws.numel()),
                                              _stream(stream)))
    return out


def tt_grad_sqnorm3(x0, x1, x2, out=None, ws=None, stream=None):
    """Sums of squares of three tensors (same dtype) in one launch -> out [3] fp64 (device)."""
    import torch
    out = torch.zeros(3, dtype=torch.float64, device=x0.device) if out is None else out
    L = lib()
    need = int(L.tt_grad_sqnorm_workspace(0))
    if ws is None or ws.numel() < need:
        ws = torch.empty(need, dtype=torch.uint8, device=x0.device)
    _check("tt_grad_sqnorm3", L.tt_grad_sqnorm3(_p(x0), int(x0.numel()), _p(x1), int(x1.numel()), _p(x2),
                                                int(x2.numel()), _dt(x0), _p(out), _p(ws), int(ws.numel()),
                                                _stream(stream)))
    return out


def tt_lmhead_loss_workspace(pk: PackedTree, hidden, vocab, vocab_chunk=16384) -> int:
    n = C.c_size_t()
    _check("tt_lmhead_loss_workspace", lib().tt_lmhead_loss_workspace(C.byref(pk.c), int(hidden), int(vocab),
                                                                      int(vocab_chunk), C.byref(n)))
    return int(n.value)


def tt_lmhead_loss(pk: PackedTree, h, w, tok, grad_scale=1.0, vocab_chunk=16384, node_loss_mask=None,
                   boundary_mode=0, dh=None, dw=None, tok_loss=None, sums=None, d_err=None, ws=None, stream=None):
    """NEXT-f3: loss + (dH, dW) of the LM head without materialising [N, V] logits.
    Returns (sums [2] fp64 device: (sum loss, sum Omega), dh, dw, tok_loss, d_err)."""
    import torch
    N, hidden = h.shape
    vocab = w.shape[0]
    dh = torch.empty_like(h) if dh is None else dh
    dw = torch.empty_like(w) if dw is None else dw
    sums = torch.zeros(2, dtype=torch.float64, device=h.device) if sums is None else sums
    d_err = torch.zeros(1, dtype=torch.int32, device=h.device) if d_err is None else d_err
    need = tt_lmhead_loss_workspace(pk, hidden, vocab, vocab_chunk)
    if ws is None or ws.numel() < need:
        ws = torch.empty(need, dtype=torch.uint8, device=h.device)
    if node_loss_mask is not None and not isinstance(node_loss_mask, torch.Tensor):
        node_loss_mask = torch.as_tensor(np.asarray(node_loss_mask, dtype=np.uint8), device=h.device)
    for t in (h, w, dh, dw):
        if not t.is_contiguous():
            raise ValueError("tensors must be contiguous")
    for t, n in ((h, "h"), (w, "w"), (dh, "dh"), (dw, "dw")):
        _need(t, torch.bfloat16, n)
    _need(tok_loss, torch.float32, "tok_loss")
    _need(sums, torch.float64, "sums")
    _need(d_err, torch.int32, "d_err")
    _need(tok, torch.int32, "tok")
    _check("tt_lmhead_loss", lib().tt_lmhead_loss(C.byref(pk.c), _p(h), _p(w), int(hidden), int(vocab),
                                                  int(vocab_chunk), _p(tok), _p(node_loss_mask), int(boundary_mode),
                                                  float(grad_scale), _p(dh), _p(dw), _p(tok_loss), _p(sums),
                                                  _p(d_err), _p(ws), int(ws.numel()), _stream(stream)))
    return sums, dh, dw, tok_loss, d_err


def tt_gemm(a, b, a_mn=False, b_mn=False, out=None, out_dtype=None, accumulate=False, stream=None):
    """D = A . B on the library's tcgen05 GEMM.  a: bf16 [M, K] (a_mn=False) or [K, M] (a_mn=True);
    b: bf16 [N, K] (b_mn=False) or [K, N] (b_mn=True); unit column stride, row stride = stride(0).
    out: [M, N] bf16 or fp32 (accumulate=True adds into an fp32 out)."""
    import torch
    for t, n in ((a, "a"), (b, "b")):
        if t.dim() != 2 or t.dtype != torch.bfloat16 or t.stride(1) != 1:
            raise ValueError(f"{n} must be a bf16 matrix with unit column stride")
    M, K = (a.shape[1], a.shape[0]) if a_mn else (a.shape[0], a.shape[1])
    N, K2 = (b.shape[1], b.shape[0]) if b_mn else (b.shape[0], b.shape[1])
    if K != K2:
        raise ValueError(f"inner dimensions differ: {K} vs {K2}")
    if out is None:
        out = torch.zeros(M, N, dtype=out_dtype or torch.float32, device=a.device)
    if out.dim() != 2 or out.shape[0] != M or out.shape[1] != N or out.stride(1) != 1:
        raise ValueError("out must be [M, N] with unit column stride")
    if b.device != a.device or out.device != a.device:
        raise ValueError("a, b, out must share a device")
    _check("tt_gemm", lib().tt_gemm(M, N, K, _p(a), a.stride(0), int(bool(a_mn)), _p(b), b.stride(0), int(bool(b_mn)),
                                    _p(out), out.stride(0), _dt(out), int(bool(accumulate)), _stream(stream)))
    return out


def tt_rope(pk: PackedTree, x, base=1.0e6, inverse=False, stream=None):
    """Rotate x [N, H, d] in place by the restored positions of pk (NEXT-f2, reading R21)."""
    if not x.is_contiguous() or x.dim() != 3:
        raise ValueError("x must be a contiguous [N, H, d] tensor")
    N, H, d = x.shape
    _check("tt_rope", lib().tt_rope(C.byref(pk.c), _p(x), _dt(x), H, d, float(base), int(bool(inverse)),
                                    _stream(stream)))
    return x


def tt_restore_grad(pk: PackedTree, g, stream=None):
    """Gradient Scaler: g[i, ...] *= tree-scale of token i, in place."""
    if not g.is_contiguous():
        raise ValueError("g must be contiguous")
    row = g.numel() // g.shape[0]
    _check("tt_restore_grad", lib().tt_restore_grad(C.byref(pk.c), _p(g), _dt(g), int(row), _stream(stream)))
    return g


def tt_plan_traversals(parent, length, capacity, term=None):
    """Capacity-constrained Tree Packing (host).  Returns (traversal id per canonical trajectory
    [n_traj] int32 numpy, info dict)."""
    par, pp = _host_i32(parent)
    ln, lp = _host_i32(length)
    tm, tp = _host_i32(term)
    info = TTPlanInfo()
    L = lib()
    _check("tt_plan_traversals", L.tt_plan_traversals(pp, lp, tp, int(par.shape[0]), int(capacity), None, C.byref(info)))
    out = np.zeros(max(info.n_traj, 1), np.int32)
    _check("tt_plan_traversals", L.tt_plan_traversals(pp, lp, tp, int(par.shape[0]), int(capacity),
                                                      out.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(info)))
    return out[:info.n_traj], {f: getattr(info, f) for f, _ in TTPlanInfo._fields_}


def tt_traversal_forest(parent, length, traversal_of_traj, traversal, term=None):
    """Sub-forest induced by one traversal -> (parent, len, term, original node ids) numpy int32."""
    par, pp = _host_i32(parent)
    ln, lp = _host_i32(length)
    tm, tp = _host_i32(term)
    tv, tvp = _host_i32(traversal_of_traj)
    n = int(par.shape[0])
    op, ol, ot, on = (np.zeros(n, np.int32) for _ in range(4))
    m = C.c_int32()
    ptr = lambda a: a.ctypes.data_as(C.POINTER(C.c_int32))
    _check("tt_traversal_forest", lib().tt_traversal_forest(pp, lp, tp, n, tvp, int(traversal), ptr(op), ptr(ol),
                                                            ptr(ot), ptr(on), C.byref(m)))
    k = m.value
    return op[:k], ol[:k], ot[:k], on[:k]
