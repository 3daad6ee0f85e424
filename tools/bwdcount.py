import ctypes, os, sys, torch
sys.path.insert(0, '/root/repo')
os.environ["TT_DEBUG_BWD"] = os.environ.get("TT_DEBUG_BWD", "8")
import paper_2511_00413_b200 as tt
from workloads import trees, tensors
L = tt.lib()
for cfg, seed in [("agentic8k", 0), ("deep32k", 1), ("wide", None)]:
    t = trees.config_tree(cfg, seed); c = trees.CONFIGS[cfg]
    pk = tt.tt_pack(t.parent, t.length); N = pk.n_tokens; hq, hkv, d = c["hq"], c["hkv"], c["d"]
    q, k, v = (x.cuda() for x in tensors.qkv_tensors(N, hq, hkv, d, "bf16", seed=0))
    G = tensors.grad_tensor(N, hq, d, "bf16", seed=1).cuda()
    o, lse = tt.tt_attn_fwd(pk, q, k, v)
    buf = (ctypes.c_ulonglong * 20)()
    tt.tt_attn_bwd(pk, q, k, v, o, lse, G); torch.cuda.synchronize()
    L.tt_debug_bwd_counters(buf, 1)
    tt.tt_attn_bwd(pk, q, k, v, o, lse, G); torch.cuda.synchronize()
    L.tt_debug_bwd_counters(buf, 1)
    b = list(buf); nit = b[4]
    print(cfg, "iters", nit, "per-iter cycles: mma_total %.0f  wait_sm %.0f  wait_dqfree %.0f  wait_q %.0f | compute(wg0,r0): wait_s %.0f  elem %.0f [ld %.0f math %.0f st %.0f] drain %.0f (wait dqfull %.0f)" %
          tuple(x / nit for x in [b[0], b[1], b[2], b[3], b[5], b[6], b[9], b[10], b[11], b[7], b[8]]), flush=True)
    ni = max(b[15], 1)
    print("   CTAs", b[13], "items", b[15], "mean CTA lifetime %.0f cycles, mean MMA-loop %.0f cycles, loop fraction %.3f, item boundary (MMA: item start -> first S/dP issued) %.0f cycles per later item" %
          (b[12] / b[13], b[0] / b[13], b[0] / b[12], b[14] / max(ni - b[13], 1)), flush=True)
    print("   item boundary waits per later item: acc_free %.0f  k_full %.0f  v_full %.0f" % tuple(x / max(ni - b[13], 1) for x in b[16:19]), flush=True)
