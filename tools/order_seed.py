"""CTA order A/B on one deep32k tree per seed (dev build: TT_BWD_CHUNK / TT_FWD_CHUNK), sustained."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_00413_b200 as tt
from workloads import trees, tensors
from tools.gemm_sustained import run

cfg, seed = sys.argv[1], int(sys.argv[2])
label = sys.argv[3] if len(sys.argv) > 3 else ""
t = trees.config_tree(cfg, seed); c = trees.CONFIGS[cfg]
pk = tt.tt_pack(t.parent, t.length)
N, hq, hkv, d = pk.n_tokens, c["hq"], c["hkv"], c["d"]
q, k, v = (x.cuda() for x in tensors.qkv_tensors(N, hq, hkv, d, "bf16", seed=0))
G = tensors.grad_tensor(N, hq, d, "bf16", seed=1).cuda()
o = torch.empty_like(q); lse = torch.empty(hq, N, device="cuda")
dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
ws = torch.empty(tt.tt_attn_bwd_workspace(pk, hq, hkv, d, q.dtype), dtype=torch.uint8, device="cuda")
A = pk.info["n_pairs"]
tt.tt_attn_fwd(pk, q, k, v, out=o, lse=lse)
run(f"{cfg}/{seed} fwd {label}", lambda: tt.tt_attn_fwd(pk, q, k, v, out=o, lse=lse), 4.0 * d * hq * A, secs=3.0)
run(f"{cfg}/{seed} bwd {label}", lambda: tt.tt_attn_bwd(pk, q, k, v, o, lse, G, dq=dq, dk=dk, dv=dv, ws=ws), 10.0 * d * hq * A, secs=3.0)
