"""Diagnose random loss sweep cases (development tool; test infrastructure)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import oracle
import paper_2511_00413_b200 as tt
from workloads import trees, tensors
import test_gpu_random_sweep as T
for seed in [int(x) for x in sys.argv[1:]]:
    t, rng = T._forest(seed + 100)
    pk = tt.tt_pack(t.parent, t.length, t.term)
    N = pk.n_tokens
    V = int(rng.choice([8, 40, 1000, 4104]))
    gamma = float(rng.choice([1.0, 0.25]))
    mask = (rng.random(len(t.parent)) < 0.8).astype(np.uint8) if seed % 2 else None
    bmode = int(seed % 4 == 3)
    x = tensors.logits_tensor(N, V, seed=seed)
    tok = tensors.token_ids(N, V, seed=seed + 1)
    tl = torch.empty(N, device="cuda", dtype=torch.float32)
    sums, dl, tl, err = tt.tt_restore_loss(pk, x.cuda(), tok.cuda(), grad_scale=gamma, node_loss_mask=mask,
                                           boundary_mode=bmode, tok_loss=tl)
    torch.cuda.synchronize()
    opk = oracle.pack(t.parent, t.length, t.term)
    lr, om, odx = oracle.loss(opk, tok.numpy(), V, np.arange(N), x, gamma=gamma, node_loss_mask=mask, boundary_mode=bmode)
    got = tl.cpu().double().numpy()
    d = np.abs(got - lr)
    tol = 1e-5 * np.abs(lr) + 1e-4 * np.maximum(om, 1).max()
    bad = np.flatnonzero(d > tol)
    print("seed", seed, "N", N, "V", V, "gamma", gamma, "mask", mask is not None, "bmode", bmode, "err", int(err.item()))
    for i in bad[:8]:
        print("   row", i, "got", got[i], "ref", lr[i], "omega", om[i], "diff", d[i], "tol", tol[i])
