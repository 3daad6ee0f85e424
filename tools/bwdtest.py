import torch, math, numpy as np, sys
sys.path.insert(0, '/root/repo')
import paper_2511_00413_b200 as tt
import oracle
from workloads import trees, tensors
def rel(a, b):
    a = a.cpu().double().numpy(); return np.linalg.norm(a - b) / np.linalg.norm(b)
for name, t, hq, hkv in [("chain128", trees.chain(1, seg=128), 1, 1), ("chain300", trees.chain(1, seg=300), 2, 1),
                         ("agentic1500", trees.gen_agentic(1500, root_len=300, seed=5), 2, 2),
                         ("gqa2000", trees.gen_agentic(2000, root_len=256, seed=1), 4, 1)]:
    pk = tt.tt_pack(t.parent, t.length)
    N = pk.n_tokens
    q, k, v = tensors.qkv_tensors(N, hq, hkv, 128, "bf16", seed=1)
    G = tensors.grad_tensor(N, hq, 128, "bf16", seed=2)
    scale = 1/math.sqrt(128)
    qd, kd, vd, Gd = q.cuda(), k.cuda(), v.cuda(), G.cuda()
    o, lse = tt.tt_attn_fwd(pk, qd, kd, vd, scale)
    dq, dk, dv = tt.tt_attn_bwd(pk, qd, kd, vd, o, lse, Gd, restore=True, softmax_scale=scale)
    torch.cuda.synchronize()
    opk = oracle.pack(t.parent, t.length)
    odq, odk, odv = oracle.attn_bwd(opk, q, k, v, G, scale)
    print(name, "dq", rel(dq, odq), "dk", rel(dk, odk), "dv", rel(dv, odv), flush=True)
