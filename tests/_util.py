"""Shared helpers for the GPU parity tests (comparison metrics and tolerances).

Tolerances (BASELINE.json north_star):
  pack / mask / position ids / weights / tile metadata : bit-exact
  O, LSE (bf16 I/O, fp32 accumulate)                   : max-abs <= 2e-2
  O, LSE (fp32 test mode)                              : max-abs <= 1e-4
  dQ, dK, dV (bf16)                                    : rel-L2 <= 3e-2 per tensor
  dQ, dK, dV (fp32 test mode)                          : rel-L2 <= 1e-4 per tensor
  loss rows / sums                                      : rel <= 1e-5 (fp32 math, fp64 sums)
  dlogits (bf16 out)                                    : |d - o| <= 2^-8 |o| + 1e-5 * gamma * Omega
"""
import numpy as np

TOL_O_BF16 = 2e-2
TOL_O_FP32 = 1e-4
TOL_G_BF16 = 3e-2
TOL_G_FP32 = 1e-4


def to64(t):
    import torch
    if isinstance(t, torch.Tensor):
        return t.detach().to("cpu", torch.float64).numpy()
    return np.asarray(t, dtype=np.float64)


def max_abs(a, b):
    a, b = to64(a), to64(b)
    return float(np.max(np.abs(a - b))) if a.size else 0.0


def rel_l2(a, b):
    a, b = to64(a), to64(b)
    den = np.linalg.norm(b.ravel())
    return float(np.linalg.norm((a - b).ravel()) / max(den, 1e-300))
