import torch, math, numpy as np, sys, time
sys.path.insert(0, '/root/repo')
import paper_2511_00413_b200 as tt
import oracle
from workloads import trees, tensors
torch.manual_seed(0)
for name, t, hq, hkv in [("chain128", trees.chain(1, seg=128), 1, 1), ("chain300", trees.chain(1, seg=300), 2, 1),
                         ("agentic1500", trees.gen_agentic(1500, root_len=300, seed=5), 2, 2)]:
    pk = tt.tt_pack(t.parent, t.length)
    N = pk.n_tokens
    q, k, v = tensors.qkv_tensors(N, hq, hkv, 128, "bf16", seed=1)
    scale = 1/math.sqrt(128)
    o, lse = tt.tt_attn_fwd(pk, q.cuda(), k.cuda(), v.cuda(), scale)
    torch.cuda.synchronize()
    opk = oracle.pack(t.parent, t.length)
    oo, ol = oracle.attn_fwd(opk, q, k, v, scale)
    err = np.abs(o.cpu().double().numpy() - oo).max(); errl = np.abs(lse.cpu().double().numpy() - ol).max()
    print(name, "O maxabs", err, "LSE maxabs", errl, flush=True)
