import ctypes, os, sys, torch
sys.path.insert(0, '/root/repo')
os.environ["TT_DEBUG_FWD"] = "8"
import paper_2511_00413_b200 as tt
from workloads import trees, tensors
L = tt.lib()
for cfg, seed in [("agentic8k", 0), ("deep32k", 1), ("wide", None)]:
    t = trees.config_tree(cfg, seed); c = trees.CONFIGS[cfg]
    pk = tt.tt_pack(t.parent, t.length); N = pk.n_tokens; hq, hkv, d = c["hq"], c["hkv"], c["d"]
    q, k, v = (x.cuda() for x in tensors.qkv_tensors(N, hq, hkv, d, "bf16", seed=0))
    buf = (ctypes.c_ulonglong * 16)()
    tt.tt_attn_fwd(pk, q, k, v); torch.cuda.synchronize(); L.tt_debug_fwd_counters(buf, 1)
    tt.tt_attn_fwd(pk, q, k, v); torch.cuda.synchronize(); L.tt_debug_fwd_counters(buf, 1)
    b = list(buf); T = b[3]; n = b[6]
    n = max(n, 1)
    print(cfg, "merged tiles", T, "per-tile cycles: mma_total %.0f wait_p %.0f wait_kv %.0f | softmax(tile0,half0,r0) tiles %d: wait_s %.0f compute %.0f (of which max-exchange barrier %.0f)" %
          (b[0] / T, b[1] / T, b[2] / T, n, b[4] / n, b[5] / n, b[7] / n), flush=True)
    print("   softmax phase ends (cumulative from S ready, per tile): tmem ld %.0f, mask+max %.0f, exp loop %.0f, total %.0f"
          % (b[9] / n, b[10] / n, b[11] / n, b[5] / n), flush=True)
    nc = max(b[13], 1); ni = max(b[15], 1)
    print("   CTAs", b[13], "items", b[15], "mean lifetime %.0f cycles, mean MMA loop %.0f, mean start->first K/V+Q ready %.0f, tiles/item %.1f, item boundary (MMA idle from item end to next first S) %.0f cycles per later item" %
          (b[12] / nc, b[0] / nc, b[8] / nc, T / ni, b[14] / max(ni - nc, 1)), flush=True)
