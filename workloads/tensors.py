"""Seeded tensor values (SURVEY.md §8(d) "Tensor values").

All draws are fp32 from torch.Generator('cpu').manual_seed(seed) and then rounded to the run
dtype, so the oracle (which upcasts exactly to fp64) and the GPU consume identical values.
Layout is "thd": [N, H, d] contiguous.
"""
from __future__ import annotations

import torch

_DT = {"fp32": torch.float32, "bf16": torch.bfloat16, "float32": torch.float32,
       "bfloat16": torch.bfloat16}


def _dtype(dt):
    return _DT[dt] if isinstance(dt, str) else dt


def qkv_tensors(n_tokens: int, hq: int, hkv: int, d: int, dtype="bf16", seed: int = 0):
    g = torch.Generator("cpu").manual_seed(seed)
    q = torch.randn(n_tokens, hq, d, generator=g, dtype=torch.float32)
    k = torch.randn(n_tokens, hkv, d, generator=g, dtype=torch.float32)
    v = torch.randn(n_tokens, hkv, d, generator=g, dtype=torch.float32)
    dt = _dtype(dtype)
    return q.to(dt).contiguous(), k.to(dt).contiguous(), v.to(dt).contiguous()


def grad_tensor(n_tokens: int, hq: int, d: int, dtype="bf16", seed: int = 1):
    """Upstream gradient G (= dO before restoration) ~ N(0,1)."""
    g = torch.Generator("cpu").manual_seed(seed)
    return torch.randn(n_tokens, hq, d, generator=g, dtype=torch.float32).to(_dtype(dtype)).contiguous()


def logits_tensor(n_tokens: int, vocab: int, seed: int = 2, dtype="bf16", scale: float = 2.0):
    g = torch.Generator("cpu").manual_seed(seed)
    x = torch.randn(n_tokens, vocab, generator=g, dtype=torch.float32) * scale
    return x.to(_dtype(dtype)).contiguous()


def token_ids(n_tokens: int, vocab: int, seed: int = 3):
    g = torch.Generator("cpu").manual_seed(seed)
    return torch.randint(0, vocab, (n_tokens,), generator=g, dtype=torch.int32)
