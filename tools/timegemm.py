"""Event-timed tt_gemm (tcgen05 CTA-pair GEMM) vs torch.matmul (cuBLAS) on the LM-head shapes, L2
flushed before every repetition.  Usage: python tools/timegemm.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2511_00413_b200 as tt


def timeit(fn, reps=10):
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.add_(1)
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    tt.lib()
    N, D, V, Vc = 8192, 4096, 151936, 16384
    g = torch.Generator(device="cuda").manual_seed(0)
    H = torch.randn(N, D, device="cuda", generator=g).to(torch.bfloat16)
    W = torch.randn(V, D, device="cuda", generator=g).to(torch.bfloat16)
    if "--lmhead-only" not in sys.argv:
        G = torch.randn(N, Vc, device="cuda", generator=g).to(torch.bfloat16)
        Wc = W[:Vc]
        Xo = torch.empty(N, V, device="cuda", dtype=torch.bfloat16)
        Xb = torch.empty(N, V, device="cuda", dtype=torch.bfloat16)
        Xc = torch.empty(N, Vc, device="cuda", dtype=torch.float32)
        Xcb = torch.empty(N, Vc, device="cuda", dtype=torch.bfloat16)
        dHo = torch.zeros(N, D, device="cuda", dtype=torch.float32)
        dHb = torch.empty(N, D, device="cuda", dtype=torch.bfloat16)
        dWo = torch.empty(Vc, D, device="cuda", dtype=torch.bfloat16)
        dWb = torch.empty(Vc, D, device="cuda", dtype=torch.bfloat16)
        shapes = [
            ("X=H W^T (full vocab, bf16 out)", lambda: tt.tt_gemm(H, W, out=Xo), lambda: torch.matmul(H, W.t(), out=Xb), 2.0 * N * V * D),
            ("X_c=H W_c^T (chunk, fp32 out)", lambda: tt.tt_gemm(H, Wc, out=Xc), lambda: torch.matmul(H, Wc.t(), out=Xcb), 2.0 * N * Vc * D),
            ("dH+=G W_c", lambda: tt.tt_gemm(G, Wc, b_mn=True, out=dHo, accumulate=True), lambda: torch.matmul(G, Wc, out=dHb), 2.0 * N * Vc * D),
            ("dW_c=G^T H", lambda: tt.tt_gemm(G, H, a_mn=True, b_mn=True, out=dWo), lambda: torch.matmul(G.t(), H, out=dWb), 2.0 * N * Vc * D),
        ]
        for name, mine, ref, fl in shapes:
            tm = timeit(mine)
            tr = timeit(ref)
            print(f"{name:34s} tt_gemm {tm:8.3f} ms {fl / tm / 1e9:8.1f} TFLOP/s   cuBLAS {tr:8.3f} ms {fl / tr / 1e9:8.1f} TFLOP/s")
        del G, Xo, Xb, Xc, Xcb
    # LM head end to end (8K rows, hidden 4096, Qwen3 vocabulary)
    from workloads import trees
    t = trees.gen_agentic(N, p_open=0.5, root_len=1024, seed=0)
    pk = tt.tt_pack(t.parent, t.length)
    tok = torch.randint(0, V, (N,), device="cuda", dtype=torch.int32)
    ws = torch.empty(tt.tt_lmhead_loss_workspace(pk, D, V, Vc), dtype=torch.uint8, device="cuda")
    dH, dW = torch.empty_like(H), torch.empty_like(W)
    reps = 1 if "--lmhead-only" in sys.argv else 5
    ms = timeit(lambda: tt.tt_lmhead_loss(pk, H, W, tok, vocab_chunk=Vc, dh=dH, dw=dW, ws=ws), reps=reps)
    fl = 8.0 * N * V * D
    print(f"tt_lmhead_loss N={N} D={D} V={V}: {ms:.3f} ms  {fl / ms / 1e9:.1f} TFLOP/s (8 N V D)")


if __name__ == "__main__":
    main()
