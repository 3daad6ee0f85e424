"""Backward kernel choice near the dispatch threshold: mean query tiles per (key block, kv head) item vs the
time of the persistent and the flat kernel (dev build; TT_BWD_FLAT forces either).  Usage: run twice, with
TT_BWD_FLAT=0 and =1."""
import os, sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2511_00413_b200 as tt
from workloads import trees, tensors


def bench(fn, iters=20, warm=3):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    st, en = torch.cuda.Event(True), torch.cuda.Event(True)
    ts = []
    for _ in range(iters):
        st.record(); fn(); en.record(); torch.cuda.synchronize(); ts.append(st.elapsed_time(en))
    ts.sort(); return ts[len(ts) // 2]


cases = [(8192, 1024, 32, 32), (8192, 1024, 32, 16), (8192, 1024, 32, 8), (16384, 2048, 32, 32),
         (16384, 2048, 32, 16), (16384, 4096, 32, 8), (32768, 4096, 32, 32)]
for N0, root, hq, hkv in cases:
    t = trees.gen_agentic(N0, p_open=0.5, root_len=root, seed=0)
    pk = tt.tt_pack(t.parent, t.length)
    N, d = pk.n_tokens, 128
    per_item = pk.c.sched_sum_nq * (hq // hkv) / pk.n_blk
    q, k, v = (x.cuda() for x in tensors.qkv_tensors(N, hq, hkv, d, "bf16", seed=0))
    G = tensors.grad_tensor(N, hq, d, "bf16", seed=1).cuda()
    o, lse = tt.tt_attn_fwd(pk, q, k, v)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    ws = torch.empty(tt.tt_attn_bwd_workspace(pk, hq, hkv, d, q.dtype), dtype=torch.uint8, device="cuda")
    tb = bench(lambda: tt.tt_attn_bwd(pk, q, k, v, o, lse, G, dq=dq, dk=dk, dv=dv, ws=ws))
    A = pk.info["n_pairs"]
    print(f"agentic{N0} root {root} {hq}/{hkv}: tiles/item {per_item:6.1f}  bwd {tb:.3f} ms ({10 * d * hq * A / tb / 1e9:.0f} TF/s)  "
          f"TT_BWD_FLAT={os.environ.get('TT_BWD_FLAT')}", flush=True)
