import torch, math, sys, time
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

for cfg, seed in [("agentic8k", 0), ("deep32k", 1), ("wide", None)]:
    t = trees.config_tree(cfg, seed); c = trees.CONFIGS[cfg]
    pk = tt.tt_pack(t.parent, t.length); N = pk.n_tokens; hq, hkv, d = c["hq"], c["hkv"], c["d"]
    q, k, v = (x.cuda() for x in tensors.qkv_tensors(N, hq, hkv, d, "bf16", seed=0))
    o = torch.empty_like(q); lse = torch.empty(hq, N, device="cuda")
    ms = bench(lambda: tt.tt_attn_fwd(pk, q, k, v, out=o, lse=lse))
    A = pk.info["n_pairs"]
    fl = 4 * d * hq * A
    print(f"{cfg}: N={N} A={A:.3e} fwd {ms:.3f} ms  eff {fl/ms/1e9:.1f} TFLOP/s", flush=True)
