"""timeall on a package root given by TT_ROOT (default /root/repo): same-box A/B of two builds."""
import os, sys
root = os.environ.get("TT_ROOT", "/root/repo")
sys.path.insert(0, root)
import torch
import paper_2511_00413_b200 as tt
from workloads import trees, tensors
assert os.path.dirname(tt.__file__).startswith(root), tt.__file__


def bench(fn, iters=20, warm=3):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    st, en = torch.cuda.Event(True), torch.cuda.Event(True)
    ts = []
    for _ in range(iters):
        st.record(); fn(); en.record(); torch.cuda.synchronize(); ts.append(st.elapsed_time(en))
    ts.sort(); return ts[len(ts)//2]


for a in sys.argv[1:]:
    cfg, seed = (a.split(":")[0], int(a.split(":")[1])) if ":" in a else (a, None)
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
    print(f"{os.path.basename(root)} {a}: fwd {tf:.3f} ms ({4*d*hq*A/tf/1e9:.0f} TF/s)  bwd {tb:.3f} ms ({10*d*hq*A/tb/1e9:.0f} TF/s)", flush=True)

if os.environ.get("TT_SUSTAINED"):
    # sustained (~3 s back to back, power-capped) bwd and fwd of each config, with clock / power
    sys.path.insert(0, "/root/repo")
    from tools.gemm_sustained import run
    for a in sys.argv[1:]:
        cfg, seed = (a.split(":")[0], int(a.split(":")[1])) if ":" in a else (a, None)
        t = trees.config_tree(cfg, seed); c = trees.CONFIGS[cfg]
        pk = tt.tt_pack(t.parent, t.length); N = pk.n_tokens; hq, hkv, d = c["hq"], c["hkv"], c["d"]
        q, k, v = (x.cuda() for x in tensors.qkv_tensors(N, hq, hkv, d, "bf16", seed=0))
        G = tensors.grad_tensor(N, hq, d, "bf16", seed=1).cuda()
        o = torch.empty_like(q); lse = torch.empty(hq, N, device="cuda")
        dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
        ws = torch.empty(tt.tt_attn_bwd_workspace(pk, hq, hkv, d, q.dtype), dtype=torch.uint8, device="cuda")
        A = pk.info["n_pairs"]
        tt.tt_attn_fwd(pk, q, k, v, out=o, lse=lse)
        run(f"{os.path.basename(root)} {a} fwd", lambda: tt.tt_attn_fwd(pk, q, k, v, out=o, lse=lse), 4.0 * d * hq * A, secs=3.0)
        run(f"{os.path.basename(root)} {a} bwd", lambda: tt.tt_attn_bwd(pk, q, k, v, o, lse, G, dq=dq, dk=dk, dv=dv, ws=ws),
            10.0 * d * hq * A, secs=3.0)
