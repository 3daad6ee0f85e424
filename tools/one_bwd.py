"""One attention forward + backward of a workload (for ncu captures): one_bwd.py <config> [seed]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_00413_b200 as tt
from workloads import trees, tensors

cfg = sys.argv[1] if len(sys.argv) > 1 else "deep32k"
seed = int(sys.argv[2]) if len(sys.argv) > 2 else None
t = trees.config_tree(cfg, seed); c = trees.CONFIGS[cfg]
pk = tt.tt_pack(t.parent, t.length); N = pk.n_tokens; hq, hkv, d = c["hq"], c["hkv"], c["d"]
q, k, v = (x.cuda() for x in tensors.qkv_tensors(N, hq, hkv, d, "bf16", seed=0))
G = tensors.grad_tensor(N, hq, d, "bf16", seed=1).cuda()
o = torch.empty_like(q); lse = torch.empty(hq, N, device="cuda")
dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
ws = torch.empty(tt.tt_attn_bwd_workspace(pk, hq, hkv, d, q.dtype), dtype=torch.uint8, device="cuda")
tt.tt_attn_fwd(pk, q, k, v, out=o, lse=lse)
tt.tt_attn_bwd(pk, q, k, v, o, lse, G, dq=dq, dk=dk, dv=dv, ws=ws)
torch.cuda.synchronize()
