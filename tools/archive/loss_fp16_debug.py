"""Worst dlogits elements of tt_restore_loss vs the oracle (small-vocabulary random case)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, paper_2511_00413_b200 as tt
from workloads import trees, tensors
t = trees.gen_agentic(600, root_len=100, seed=3)
V, gamma = 1000, 0.5
pk = tt.tt_pack(t.parent, t.length)
N = pk.n_tokens
x = tensors.logits_tensor(N, V, seed=0)
tok = tensors.token_ids(N, V, seed=1)
sums, dl, _, err = tt.tt_restore_loss(pk, x.cuda(), tok.cuda(), grad_scale=gamma)
torch.cuda.synchronize()
opk = oracle.pack(t.parent, t.length)
lr, om, dx = oracle.loss(opk, tok.numpy(), V, np.arange(N), x, gamma=gamma)
g = dl.cpu().double().numpy()
tol = 2.0 ** -8 * np.abs(dx) + 1e-5 * abs(gamma) * np.maximum(om, 1.0)[:, None]
bad = np.argwhere(np.abs(g - dx) > tol)
print("bad elements", len(bad), "rows", len(set(bad[:, 0])) if len(bad) else 0)
for r, c in bad[:20]:
    print(r, c, "got", g[r, c], "ref", dx[r, c], "omega", om[r], "x", float(x[r, c]), "rel", abs(g[r, c] - dx[r, c]) / abs(dx[r, c]))
