import torch, sys
sys.path.insert(0, '/root/repo')
import paper_2511_00413_b200 as tt
from workloads import trees
for cfg, seed in [(c, 0 if c != "wide" else None) for c in (sys.argv[1:] or ["agentic8k", "wide"])]:
    t = trees.config_tree(cfg, seed); pk = tt.tt_pack(t.parent, t.length); N = pk.n_tokens; V = 151936
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.empty(N, V, device="cuda", dtype=torch.bfloat16)
    for r0 in range(0, N, 2048): x[r0:r0+2048] = (2*torch.randn(min(2048, N-r0), V, device="cuda", generator=g)).bfloat16()
    tok = torch.randint(0, V, (N,), device="cuda", dtype=torch.int32, generator=g)
    dl = torch.empty_like(x); fl = torch.empty(64*1024*1024, device="cuda")
    ts = []
    for i in range(8):
        fl.add_(1); a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); tt.tt_restore_loss(pk, x, tok, dlogits=dl); b.record(); torch.cuda.synchronize()
        if i >= 3: ts.append(a.elapsed_time(b))
    ms = sorted(ts)[len(ts)//2]
    print(f"{cfg}: loss {ms:.3f} ms  {N*(4*V+12)/ms/1e6:.0f} GB/s", flush=True)
