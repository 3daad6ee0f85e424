"""B200 (sm_100a) hot path of Tree Training (arXiv 2511.00413).

The compute lives in libtt.so (hand-written CUDA for sm_100a behind the C ABI of include/tt.h);
this package is a thin ctypes binding with the same names.  PyTorch is used only for device
memory, streams and process groups.  There is no CPU fallback: if libtt.so is missing or cannot be
loaded, importing the binding raises.
"""
from .binding import (  # noqa: F401
    TTError, PackedTree, lib, lib_path, tt_pack_plan, tt_pack, tt_pack_weights, tt_attn_fwd, tt_attn_bwd,
    tt_attn_bwd_workspace, tt_attn_bwd_kernel, tt_restore_loss, tt_grad_sqnorm, tt_grad_sqnorm3, tt_launch_count, tt_launch_count_reset,
    tt_plan_traversals, tt_traversal_forest, tt_rope, tt_restore_grad, tt_lmhead_loss,
    tt_lmhead_loss_workspace, tt_gemm, TT_BLOCK,
)

__all__ = ["TTError", "PackedTree", "lib", "lib_path", "tt_pack_plan", "tt_pack", "tt_pack_weights", "tt_attn_fwd",
           "tt_attn_bwd", "tt_attn_bwd_workspace", "tt_attn_bwd_kernel", "tt_restore_loss", "tt_grad_sqnorm", "tt_grad_sqnorm3",
           "tt_launch_count", "tt_launch_count_reset", "tt_plan_traversals", "tt_traversal_forest", "tt_rope",
           "tt_restore_grad", "tt_lmhead_loss", "tt_lmhead_loss_workspace", "TT_BLOCK"]
