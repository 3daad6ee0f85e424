"""Diagnose tt_lmhead_loss after the attention tests have run (development tool)."""
import sys, subprocess
import numpy as np
import torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import pytest
rc = pytest.main(["-x", "-q", "-m", "gpu", sys.argv[1]] if len(sys.argv) > 1 else ["-x", "-q", "-m", "gpu", "tests/test_gpu_attn.py"])
import paper_2511_00413_b200 as tt
import oracle
from oracle import lmhead as ol
from workloads import trees
t = trees.gen_agentic(700, root_len=150, seed=3)
pk = tt.tt_pack(t.parent, t.length)
N, D, V = pk.n_tokens, 256, 5003
g = torch.Generator().manual_seed(11)
H = torch.randn(N, D, generator=g).to(torch.bfloat16)
W = (2.0 / D ** 0.5 * torch.randn(V, D, generator=g)).to(torch.bfloat16)
tok = torch.randint(0, V, (N,), generator=g, dtype=torch.int32)
opk = oracle.pack(t.parent, t.length)
r = ol.lmhead_loss(opk, H.double().numpy(), W.double().numpy(), tok.numpy())
for it in range(3):
    tl = torch.empty(N, device="cuda")
    sums, dh, dw, tl, err = tt.tt_lmhead_loss(pk, H.cuda(), W.cuda(), tok.cuda(), vocab_chunk=1024, tok_loss=tl)
    torch.cuda.synchronize()
    v = tl.cpu().double().numpy()
    d = np.abs(v - r["loss_rows"])
    badr = np.flatnonzero(d > 1e-3 * np.maximum(1, np.abs(r["loss_rows"])))
    print("iter", it, "err", int(err.item()), "bad rows", len(badr), badr[:20], v[badr[:5]], r["loss_rows"][badr[:5]], flush=True)
    # materialised check of the chunk GEMM
    X = (H.cuda().float() @ W.cuda().float().T)
    print("  torch lse row0", float(torch.logsumexp(X[0], 0)), flush=True)
