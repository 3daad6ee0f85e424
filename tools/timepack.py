"""Host-side cost of tt_pack on the bench tree (development tool): wall time of the binding call and
its pieces, and the CUDA-event window the bench's "pack" op sees."""
import sys
import time
import ctypes as C
sys.path.insert(0, "/root/repo")
import torch
import paper_2511_00413_b200 as tt
from paper_2511_00413_b200 import binding as B
from workloads import trees

t = trees.config_tree("agentic8k", 0)
L = B.lib()
for _ in range(20):
    tt.tt_pack(t.parent, t.length)
torch.cuda.synchronize()
n = 200
t0 = time.perf_counter()
for _ in range(n):
    tt.tt_pack(t.parent, t.length)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"tt_pack binding call: {(t1 - t0) / n * 1e6:.1f} us wall per call")
par, pp = B._host_i32(t.parent); ln, lp = B._host_i32(t.length); tm, tp = B._host_i32(t.term)
info = B.TTPackInfo()
t0 = time.perf_counter()
for _ in range(n):
    L.tt_pack_plan(pp, lp, tp, int(par.shape[0]), C.byref(info))
print(f"tt_pack_plan: {(time.perf_counter() - t0) / n * 1e6:.1f} us")
t0 = time.perf_counter()
for _ in range(n):
    ws = torch.empty(int(info.ws_bytes) + 256, dtype=torch.uint8, device="cuda")
print(f"torch.empty ws: {(time.perf_counter() - t0) / n * 1e6:.1f} us")
c = B.TTPacked(); info2 = B.TTPackInfo()
ws = torch.empty(int(info.ws_bytes) + 256, dtype=torch.uint8, device="cuda")
base = ws.data_ptr() + ((-ws.data_ptr()) % 256)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(n):
    L.tt_pack(pp, lp, tp, int(par.shape[0]), C.c_void_p(base), int(info.ws_bytes), C.byref(c), C.byref(info2),
              B._stream(None))
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"tt_pack C call: {(t1 - t0) / n * 1e6:.1f} us")
ts = []
for _ in range(20):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record(); tt.tt_pack(t.parent, t.length); b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) * 1e3)
ts.sort()
print(f"event window (idle GPU before): median {ts[len(ts)//2]:.1f} us, min {ts[0]:.1f} us")
