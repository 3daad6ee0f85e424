"""Sustained restoration loss (~3 s back to back) on one workload at V = 151,936, with the SM clock and
board power nvidia-smi saw (is the loss itself power-capped?).  Usage: loss_power.py <config> [label]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_00413_b200 as tt
from workloads import trees, tensors
from tools.gemm_sustained import run


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "deep32k"
    label = sys.argv[2] if len(sys.argv) > 2 else ""
    tt.lib()
    t = trees.config_tree(cfg)
    c = trees.CONFIGS[cfg]
    pk = tt.tt_pack(t.parent, t.length)
    N, V = pk.n_tokens, 151936
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.empty(N, V, device="cuda", dtype=torch.bfloat16)
    for r0 in range(0, N, 2048):
        x[r0:r0 + 2048] = (2 * torch.randn(min(2048, N - r0), V, device="cuda", generator=g)).bfloat16()
    tok = torch.randint(0, V, (N,), device="cuda", dtype=torch.int32, generator=g)
    bytes_per = N * (4 * V + 12)
    # run() prints "work per second / 1e12": with bytes as the work unit that column is TB/s
    run(f"{cfg} loss alone {label} [TB/s]", lambda: tt.tt_restore_loss(pk, x, tok, dlogits=x), bytes_per, secs=3.0)


if __name__ == "__main__":
    main()
