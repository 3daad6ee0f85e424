"""Which libcublasLt does libtt bind to, and does tt_lmhead_loss agree with torch there (dev tool)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
order = sys.argv[1]
if order == "torch_first":
    a = torch.randn(64, 64, device="cuda", dtype=torch.bfloat16)
    (a @ a).sum().item()
import paper_2511_00413_b200 as tt
tt.lib()
from workloads import trees
t = trees.gen_agentic(700, root_len=150, seed=3)
pk = tt.tt_pack(t.parent, t.length)
N, D, V = pk.n_tokens, 256, 5003
g = torch.Generator().manual_seed(11)
H = torch.randn(N, D, generator=g).to(torch.bfloat16).cuda()
W = (2.0 / D ** 0.5 * torch.randn(V, D, generator=g)).to(torch.bfloat16).cuda()
tok = torch.randint(0, V, (N,), generator=g, dtype=torch.int32).cuda()
tl = torch.empty(N, device="cuda")
sums, dh, dw, tl, err = tt.tt_lmhead_loss(pk, H, W, tok, vocab_chunk=1024, tok_loss=tl)
torch.cuda.synchronize()
X = H.float() @ W.float().T
print(order, "lse row0 torch", float(torch.logsumexp(X[0], 0)), "tok_loss[0:3]", tl[:3].tolist(), "sum", float(sums[0]))
for ln in open("/proc/self/maps"):
    if "cublasLt" in ln and "r-xp" in ln:
        print("  ", ln.split()[-1])
