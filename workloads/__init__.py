"""Seeded synthetic workloads shared by the oracle tests, the GPU parity tests and bench.py.

This package holds NO arithmetic of the method (no packing, no mask, no attention, no loss):
it only draws tree *shapes* (parent array + per-node token counts) and tensor *values*.
Both sides of every parity test consume exactly these arrays; neither side's code lives here.

Recipe:
  * trees: `gen_agentic` (branching factor 2-4, depth 6, lognormal segment lengths) for the
    agentic / deep configs, `gen_wide` for the 4K-prefix + 64-leaf config, `tiny` for config 1.
  * tensors: Q, K, V, G(=dO) ~ N(0,1) drawn in fp32 from torch.Generator('cpu').manual_seed(seed),
    then rounded to the run dtype; logits ~ 2*N(0,1) -> bf16; token ids ~ U[0, V).
"""
from .trees import (Tree, tiny, spec_example, fig4_unit, chain, star, gen_agentic, gen_deep,
                    gen_wide, gen_random_forest, path_token_total, config_tree, CONFIGS)
from .tensors import qkv_tensors, grad_tensor, logits_tensor, token_ids

__all__ = ["Tree", "tiny", "spec_example", "fig4_unit", "chain", "star", "gen_agentic", "gen_deep",
           "gen_wide", "gen_random_forest", "path_token_total", "config_tree", "CONFIGS",
           "qkv_tensors", "grad_tensor", "logits_tensor", "token_ids"]
