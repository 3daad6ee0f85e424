"""Stress tt_lmhead_loss: repeated calls with the caching allocator's free memory filled with garbage
in between; every call must give bitwise-identical loss rows (development tool)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
import paper_2511_00413_b200 as tt
from workloads import trees
t = trees.gen_agentic(700, root_len=150, seed=3)
pk = tt.tt_pack(t.parent, t.length)
N, D, V = pk.n_tokens, 256, 5003
g = torch.Generator().manual_seed(11)
H = torch.randn(N, D, generator=g).to(torch.bfloat16).cuda()
W = (2.0 / D ** 0.5 * torch.randn(V, D, generator=g)).to(torch.bfloat16).cuda()
tok = torch.randint(0, V, (N,), generator=g, dtype=torch.int32).cuda()
ref = None
bad = 0
for it in range(30):
    junk = torch.full((64 * 1024 * 1024,), 3.0e30 if it % 2 else float("nan"), device="cuda")
    del junk
    tl = torch.empty(N, device="cuda")
    sums, dh, dw, tl, err = tt.tt_lmhead_loss(pk, H, W, tok, vocab_chunk=1024, tok_loss=tl)
    torch.cuda.synchronize()
    v = tl.cpu().numpy()
    if ref is None:
        ref = v
    elif not np.array_equal(v, ref, equal_nan=True):
        bad += 1
        d = np.abs(v - ref)
        print("iter", it, "mismatch rows", int((d > 0).sum()), "max", float(np.nanmax(d)), flush=True)
print("bad", bad, "of 30; loss sum", float(ref.sum()), flush=True)
