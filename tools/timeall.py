import torch, math, sys
sys.path.insert(0, '/root/repo')
import paper_2511_00413_b200 as tt
from workloads import trees, tensors

def bench(fn, iters=20, warm=3):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    st, en = torch.cuda.Event(True), torch.cuda.Event(True)
    ts = []
    for _ in range(iters):
        st.record(); fn(); en.record(); torch.cuda.synchronize(); ts.append(st.elapsed_time(en))
    ts.sort(); return ts[len(ts)//2]

cfgs = [("agentic8k", 0), ("deep32k", 1), ("wide", None)] if len(sys.argv) < 2 else \
    [(a.split(":")[0], int(a.split(":")[1]) if ":" in a else None) for a in sys.argv[1:]]  # config[:seed]
for cfg, seed in cfgs:
    t = trees.config_tree(cfg, seed); c = trees.CONFIGS[cfg]
    pk = tt.tt_pack(t.parent, t.length); N = pk.n_tokens; hq, hkv, d = c["hq"], c["hkv"], c["d"]
    q, k, v = (x.cuda() for x in tensors.qkv_tensors(N, hq, hkv, d, "bf16", seed=0))
    G = tensors.grad_tensor(N, hq, d, "bf16", seed=1).cuda()
    o = torch.empty_like(q); lse = torch.empty(hq, N, device="cuda")
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    ws = torch.empty(tt.tt_attn_bwd_workspace(pk, hq, hkv, d, q.dtype), dtype=torch.uint8, device="cuda")
    tf = bench(lambda: tt.tt_attn_fwd(pk, q, k, v, out=o, lse=lse))
    tb = bench(lambda: tt.tt_attn_bwd(pk, q, k, v, o, lse, G, dq=dq, dk=dk, dv=dv, ws=ws))
    A = pk.info["n_pairs"]
    print(f"{cfg}: N={N} fwd {tf:.3f} ms ({4*d*hq*A/tf/1e9:.0f} TF/s)  bwd {tb:.3f} ms ({10*d*hq*A/tb/1e9:.0f} TF/s)  "
          f"fwd+bwd {14*d*hq*A/(tf+tb)/1e9:.0f} TF/s", flush=True)
