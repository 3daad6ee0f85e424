"""Sustained (power-capped) tt_gemm vs cuBLAS: each runs back to back for ~4 s on the LM-head chunk
shape; TFLOP/s over the window and the SM clock / power nvidia-smi saw during it."""
import os, subprocess, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_00413_b200 as tt


def smi_sampler(stop, out):
    p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                          "-lms", "100"], stdout=subprocess.PIPE, text=True)
    while not stop.is_set():
        ln = p.stdout.readline()
        if ln:
            out.append([float(x) for x in ln.split(",")])
    p.terminate()


def run(name, fn, fl, secs=4.0):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    stop, samples = threading.Event(), []
    th = threading.Thread(target=smi_sampler, args=(stop, samples), daemon=True)
    th.start()
    time.sleep(0.3)
    n, t0 = 0, time.time()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    while time.time() - t0 < secs:
        for _ in range(10):
            fn()
        n += 10
        torch.cuda.synchronize()
    b.record()
    torch.cuda.synchronize()
    stop.set()
    ms = a.elapsed_time(b)
    s = sorted(samples[len(samples) // 4:]) if samples else [[0, 0]]
    clk = sorted(x[0] for x in samples[len(samples) // 4:]) or [0]
    pw = sorted(x[1] for x in samples[len(samples) // 4:]) or [0]
    print(f"{name:28s} {n * fl / (ms * 1e-3) / 1e12:8.1f} TFLOP/s sustained  sm {clk[len(clk) // 2]:.0f} MHz  power {pw[len(pw) // 2]:.0f} W",
          flush=True)
    time.sleep(2.0)


def main():
    tt.lib()
    N, D, Vc = 8192, 4096, 16384
    g = torch.Generator(device="cuda").manual_seed(0)
    H = torch.randn(N, D, device="cuda", generator=g).to(torch.bfloat16)
    W = torch.randn(Vc, D, device="cuda", generator=g).to(torch.bfloat16)
    Xb = torch.empty(N, Vc, device="cuda", dtype=torch.bfloat16)
    fl = 2.0 * N * Vc * D
    tag = os.environ.get("TT_GEMM_WAIT", "-")
    run(f"tt_gemm H W^T wait={tag}", lambda: tt.tt_gemm(H, W, out=Xb), fl)
    if "--cublas" in sys.argv:
        run("cuBLAS  H W^T (bf16 out)", lambda: torch.matmul(H, W.t(), out=Xb), fl)


if __name__ == "__main__":
    main()
