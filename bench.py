#!/usr/bin/env python
"""bench.py — Tree Training hot path on B200: one JSON line per run (driver contract).

A "step" is one pass of the whole hot path of SURVEY.md §8(a) over the rank's trees:
  a1 tt_pack (host DFS + device fill/tile lists)   a2 tt_attn_fwd   a3 tt_restore_loss (+ loss sums)
  a4+a5 tt_attn_bwd (preprocess + main + dQ convert)   a6 ||dQ||^2, ||dK||^2, ||dV||^2 fused into
  tt_attn_bwd (per-CTA partials, fixed-order fp64 sum) + one all_gather of the per-tree fp64
  records, summed in tree-id order (NCCL at N > 1).
Default workload: BASELINE.json configs[4] "batch of 64 independent trees (64K tokens each)
sharded over 1/2/4/8 B200 with NCCL loss/grad-norm reduce" — the largest configuration, the only one
named for the 1..8-GPU curve (32 q / 8 kv heads, d 128, bf16, Qwen3-shaped attention P:562-564),
with the Gradient-Restoration loss at the Qwen3 vocabulary (151,936).  The 64 trees are
partitioned over the ranks by greedy LPT on their ancestor pairs (strong scaling: the job is fixed).
`--config agentic8k | deep32k | wide | wide_aligned` runs one tree per rank (seed = rank, weak).

value = effective attention FLOPs of the step (14 d Hq A per tree, A = ancestor pairs, i.e.
only unmasked pairs count) summed over all trees / (max over ranks of the device-timed step time).
Timing: W untimed warm-up steps, then K steps each bracketed by CUDA events on the launching
stream, L2 flushed (256 MiB write) between steps outside the events, barrier + synchronize around
the whole timed loop, max over ranks.

`--impl reference` times the fp64 CPU oracle (oracle/) on the same workload/metric: each step is a
bounded sample of the workload (heads x first trajectories of tree 0); value = the sample's share of
the effective FLOPs / its measured time, ms_per_step = the measured sample time.

Besides the driver-contract keys the line carries: per_op_ms (+ median / min), attn_fwd_bwd_tflops,
roofline (dominant kernel: algorithmic work per launch / event-timed duration vs MEASURED_PEAKS,
ncu DRAM bytes and the raw tensor-core utilisation from profiles/ncu_traffic.json) and
roofline_<fwd|loss|pack>, totals (the reduced per-tree scalars),
speedup_vs_linear (the same kernels on every trajectory linearised: attention vs the pair ratio,
the loss vs the token ratio, both together), next_f1_planner, next_f2 (RoPE / Gradient Scaler
GB/s), next_f3_lmhead (LM head + loss TFLOP/s), cpu_baseline (N = 1).  --no-linear / --no-e2e /
--no-cpu / --no-lmhead / --no-loss skip legs (profiling runs).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "tree-attn fwd+bwd effective TFLOP/s & % BF16 peak; speedup vs per-branch linear"
LOSS_KERNELS = ("loss_cluster_kernel", "loss_pipe_kernel")
VOCAB = 151936


def refuse_dev_build(tt):
    """A development build (-DTT_DEV) reads A/B switches that skip work: never time it."""
    if tt.lib().tt_build_flags() & 1:
        raise SystemExit("bench.py: libtt.so is a development build (TT_DEV); rebuild with "
                         "`python -m paper_2511_00413_b200.build --force`")


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return dict(bf16=float(d["bf16_tflops"]), bf16_sustained=float(d.get("bf16_tflops_sustained", d["bf16_tflops"])),
                    hbm=float(d["hbm_gbs"]), source="measured (MEASURED_PEAKS.json)")
    return dict(bf16=1590.0, bf16_sustained=1400.0, hbm=6650.0, source="fallback (B200_PROFILING.md)")


# ------------------------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, val in zip(names, f[4:8]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------------------------ workload
def make_trees(args, rank, world):
    from workloads import trees
    if args.config == "batch64k":
        from paper_2511_00413_b200 import sharding, tt_pack_plan
        all_trees = [trees.config_tree("batch64k", s) for s in range(args.trees)]
        work = [tt_pack_plan(t.parent, t.length)["n_pairs"] for t in all_trees]
        assign, imb = sharding.lpt_partition(work, world)   # greedy LPT, deterministic
        return [(i, all_trees[i]) for i in assign[rank]], {"lpt_imbalance": round(imb, 4)}
    seed = rank if args.seed is None else args.seed
    if args.config in ("wide", "wide_aligned"):
        return [(rank, trees.config_tree(args.config))], {}  # one shape; inputs seeded by rank
    return [(seed, trees.config_tree(args.config, seed))], {}


class Scratch:
    """Per-rank buffers shared by the trees a rank processes one after another (allocated once at
    the largest tree, untimed): outputs, logits / dlogits, the bwd workspace, pinned host buffers.
    The logits buffer is seeded by a constant (not the rank), so tree t's loss is the same value
    whichever rank processes it."""

    def __init__(self, maxN, cfg, vocab, with_loss, host_copy):
        import torch
        dev, dt = "cuda", torch.bfloat16
        hq, hkv, d = cfg["hq"], cfg["hkv"], cfg["d"]
        self.o = torch.empty(maxN, hq, d, device=dev, dtype=dt)
        self.lse = torch.empty(hq * maxN, device=dev)
        self.dq = torch.empty(maxN, hq, d, device=dev, dtype=dt)
        self.dk = torch.empty(maxN, hkv, d, device=dev, dtype=dt)
        self.dv = torch.empty(maxN, hkv, d, device=dev, dtype=dt)
        self.ws = None
        if with_loss:
            gen = torch.Generator(device=dev).manual_seed(4242)
            self.logits = torch.empty(maxN, vocab, device=dev, dtype=dt)
            for r0 in range(0, maxN, 2048):  # chunked to bound the fp32 temporary
                r1 = min(maxN, r0 + 2048)
                self.logits[r0:r1] = (2.0 * torch.randn(r1 - r0, vocab, device=dev, generator=gen)).to(dt)
            self.dlogits = torch.empty_like(self.logits)
            self.tok_loss = torch.empty(maxN, device=dev)
        self.host = None
        if host_copy:
            # pinned host sources of one tree's step inputs (re-used for every tree of the rank: the
            # bytes each tree copies are its own N rows) and pinned destinations of its gradients
            hg = torch.Generator().manual_seed(99)
            self.host = {n: torch.randn(maxN, h, d, generator=hg).to(dt).pin_memory()
                         for n, h in (("q", hq), ("k", hkv), ("v", hkv), ("g", hq))}
            if with_loss:
                self.host["logits"] = self.logits.cpu().pin_memory()
                self.host["tok"] = torch.randint(0, vocab, (maxN,), generator=hg, dtype=torch.int32).pin_memory()
            self.host_out = {"dq": torch.empty(maxN, hq, d, dtype=dt).pin_memory(),
                             "dk": torch.empty(maxN, hkv, d, dtype=dt).pin_memory(),
                             "dv": torch.empty(maxN, hkv, d, dtype=dt).pin_memory()}


class TreeJob:
    """Device-resident inputs for one tree (allocated once, untimed), drawn from a generator seeded
    by the tree id (the same tensors whichever rank processes the tree); outputs live in the rank's
    shared Scratch (trees of a rank run one after another)."""

    def __init__(self, tid, tree, cfg, vocab, scratch, with_loss=True, host_copy=False):
        import torch
        import paper_2511_00413_b200 as tt
        self.tid, self.tree = tid, tree
        self.hq, self.hkv, self.d = cfg["hq"], cfg["hkv"], cfg["d"]
        info = tt.tt_pack_plan(tree.parent, tree.length)
        self.info = info
        N = self.N = info["n_tokens"]
        dt = torch.bfloat16
        dev = "cuda"
        gen = torch.Generator(device=dev).manual_seed(1_000_003 + int(tid))
        self.q = torch.randn(N, self.hq, self.d, device=dev, dtype=torch.float32, generator=gen).to(dt)
        self.k = torch.randn(N, self.hkv, self.d, device=dev, dtype=torch.float32, generator=gen).to(dt)
        self.v = torch.randn(N, self.hkv, self.d, device=dev, dtype=torch.float32, generator=gen).to(dt)
        self.g = torch.randn(N, self.hq, self.d, device=dev, dtype=torch.float32, generator=gen).to(dt)
        S = self.scratch = scratch
        self.o, self.dq, self.dk, self.dv = S.o[:N], S.dq[:N], S.dk[:N], S.dv[:N]
        self.lse = S.lse[:self.hq * N].view(self.hq, N)
        self.with_loss = with_loss
        self.vocab = vocab
        if with_loss:
            self.logits, self.dlogits, self.tok_loss = S.logits[:N], S.dlogits[:N], S.tok_loss[:N]
            self.tok = torch.randint(0, vocab, (N,), device=dev, dtype=torch.int32, generator=gen)
            self.err = torch.zeros(1, dtype=torch.int32, device=dev)
        self.rec = torch.zeros(5, dtype=torch.float64, device=dev)
        self.host = None
        if host_copy:
            self.host = {n: t[:N] for n, t in S.host.items()}
            self.host_out = {n: t[:N] for n, t in S.host_out.items()}
            self.rec_host = torch.zeros(5, dtype=torch.float64).pin_memory()

    @property
    def ws(self):
        return self.scratch.ws

    @ws.setter
    def ws(self, value):
        self.scratch.ws = value

    def flops(self):
        return 14.0 * self.d * self.hq * self.info["n_pairs"]

    def h2d_bytes(self):
        return sum(t.numel() * t.element_size() for t in self.host.values()) if self.host else 0

    def d2h_bytes(self):
        return (sum(t.numel() * t.element_size() for t in self.host_out.values()) + 40) if self.host else 0


def run_step(job, ev=None, h2d=False):
    """One pass of the hot path for one tree.  ev: dict of event pairs for per-op timing.  h2d: the
    end-to-end form — inputs copied in from pinned host memory first, the gradients dQ / dK / dV and
    the tree's scalar record copied back after (dlogits stays on the device, where the LM-head
    backward consumes it)."""
    import torch
    import paper_2511_00413_b200 as tt

    def mark(name, i):
        if ev is not None:
            ev[name][i].record()

    if h2d:
        for n, t in job.host.items():
            getattr(job, n).copy_(t, non_blocking=True)
    mark("pack", 0)
    pk = tt.tt_pack(job.tree.parent, job.tree.length)                                   # a1
    mark("pack", 1)
    mark("fwd", 0)
    tt.tt_attn_fwd(pk, job.q, job.k, job.v, out=job.o, lse=job.lse)                      # a2
    mark("fwd", 1)
    if job.with_loss:
        mark("loss", 0)
        tt.tt_restore_loss(pk, job.logits, job.tok, grad_scale=1.0, dlogits=job.dlogits,   # a3
                           tok_loss=job.tok_loss, sums=job.rec[0:2], d_err=job.err)
        mark("loss", 1)
    need = tt.tt_attn_bwd_workspace(pk, job.hq, job.hkv, job.d, job.q.dtype)
    if job.ws is None or job.ws.numel() < need:
        job.ws = torch.empty(need, dtype=torch.uint8, device="cuda")
    mark("bwd", 0)
    tt.tt_attn_bwd(pk, job.q, job.k, job.v, job.o, job.lse, job.g, restore=True,          # a4 + a5 (+ a6:
                   dq=job.dq, dk=job.dk, dv=job.dv, ws=job.ws, sqnorm=job.rec[2:5])       # fused norms)
    mark("bwd", 1)
    if h2d:
        for n, t in job.host_out.items():
            t.copy_(getattr(job, n), non_blocking=True)
        job.rec_host.copy_(job.rec, non_blocking=True)
    return pk


def aggregate(records, my_ms, my_flops, n_trees, dist_mod=None, world=1, device=None):
    """The step's cross-rank aggregation, shared by the timed run and the CPU tests:
    one all_gather_into_tensor of the fixed-size per-tree fp64 records [tree id, sum loss, sum Omega,
    |dQ|^2, |dK|^2, |dV|^2], summed in tree-id order on every rank (so each total is a function of
    the per-tree records alone, whatever the world size), and the job time = max over ranks of the
    device-timed rank time, FLOPs summed over ranks.  records: list of (tree id, 5 values).
    Returns (totals [5], n_trees seen, max ms, total FLOPs)."""
    import torch
    from paper_2511_00413_b200 import sharding
    slot = sharding.pack_records(records, n_trees, world, device=device)
    if world > 1:
        gathered = sharding.gather_records(slot, dist_mod, world)
        tv = torch.tensor([my_ms, my_flops], dtype=torch.float64, device=device)
        allv = torch.empty(2 * world, dtype=torch.float64, device=device)
        dist_mod.all_gather_into_tensor(allv, tv)
        allv = allv.view(world, 2).cpu()
        t_max, flops = float(allv[:, 0].max()), float(allv[:, 1].sum())
    else:
        gathered, t_max, flops = slot, float(my_ms), float(my_flops)
    tot, n = sharding.reduce_records(gathered)
    return tot, n, t_max, flops


def _longest_paths(tree):
    """Token length of every root-to-node path that ends a trajectory (plain parent walk)."""
    par, ln = tree.parent, tree.length
    has_child = np.zeros(len(par), bool)
    has_child[par[par >= 0]] = True
    ends = np.flatnonzero(~has_child) if tree.term is None else np.flatnonzero(tree.term > 0)
    for v in ends:
        s, u = 0, int(v)
        while u >= 0:
            s += int(ln[u])
            u = int(par[u])
        yield s


def flush_l2(buf):
    buf.add_(1)  # 256 MiB read+write > 126 MB L2


# ------------------------------------------------------------------------------------ linear
def trajectory_token_paths(pk, tree):
    """Packed token indices of every root-to-leaf trajectory (childless nodes, or term copies),
    from the product pack's own node_start / node_len (no oracle on this leg): the comparison input
    of the per-branch linear runs."""
    arr = pk.arrays()
    start = arr["node_start"].cpu().numpy().astype(np.int64)
    nlen = arr["node_len"].cpu().numpy().astype(np.int64)
    par = np.asarray(tree.parent, dtype=np.int64)
    n = len(par)
    has_child = np.zeros(n, bool)
    has_child[par[par >= 0]] = True
    term = (~has_child).astype(np.int64) if tree.term is None else np.asarray(tree.term, dtype=np.int64)
    ends = [v for v in range(n) for _ in range(int(term[v]))]
    ends.sort(key=lambda v: (start[v], v))  # DFS pre-order of the end nodes
    paths = []
    for v in ends:
        chain, u = [], v
        while u >= 0:
            chain.append(u)
            u = int(par[u])
        paths.append(np.concatenate([np.arange(start[u], start[u] + nlen[u]) for u in reversed(chain)]
                                    + [np.zeros(0, np.int64)]))
    return paths


def linear_attention_time(job, reps=5, tree_only=False):
    """Same kernels on the linearised forest (every root-to-leaf trajectory as its own root;
    untimed gather).  Returns (fwd+bwd ms, linear pairs, linear tokens).  tree_only: the tree's own
    fwd + bwd time under the same protocol (returns ms)."""
    import torch
    import paper_2511_00413_b200 as tt
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    if tree_only:
        pk = tt.tt_pack(job.tree.parent, job.tree.length, job.tree.term)
        lq, lk, lv, lg, o, lse, dq, dk, dv = job.q, job.k, job.v, job.g, job.o, job.lse, job.dq, job.dk, job.dv
        restore = True
    else:
        paths = trajectory_token_paths(tt.tt_pack(job.tree.parent, job.tree.length, job.tree.term), job.tree)
        idx = torch.as_tensor(np.concatenate(paths).astype(np.int64), device="cuda")
        lens = [len(p) for p in paths]
        lq, lk, lv, lg = (x.index_select(0, idx).contiguous() for x in (job.q, job.k, job.v, job.g))
        pk = tt.tt_pack([-1] * len(lens), lens)
        o = torch.empty_like(lq)
        lse = torch.empty(job.hq, pk.n_tokens, device="cuda")
        dq, dk, dv = torch.empty_like(lq), torch.empty_like(lk), torch.empty_like(lv)
        restore = False
    ws = torch.empty(tt.tt_attn_bwd_workspace(pk, job.hq, job.hkv, job.d, lq.dtype), dtype=torch.uint8, device="cuda")
    ts = []
    for r in range(reps + 2):
        flush_l2(flush)
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        tt.tt_attn_fwd(pk, lq, lk, lv, out=o, lse=lse)
        tt.tt_attn_bwd(pk, lq, lk, lv, o, lse, lg, restore=restore, dq=dq, dk=dk, dv=dv, ws=ws)
        b.record()
        torch.cuda.synchronize()
        if r >= 2:
            ts.append(a.elapsed_time(b))
    if tree_only:
        return float(np.median(ts))
    return float(np.median(ts)), pk.info["n_pairs"], pk.info["n_tokens"]


def linear_loss_time(job, max_rows=32768, reps=3, tree_only=False):
    """The Gradient-Restoration loss kernel on the linearised rows: every trajectory as its own root
    (w = 1), processed in chunks of whole trajectories (<= max_rows rows) through one in-place logits
    buffer (dlogits aliases logits), chunk times summed.  Returns (ms, linear rows).  tree_only: the
    tree's own loss launch under the same protocol."""
    import torch
    import paper_2511_00413_b200 as tt
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    if tree_only:
        pk = tt.tt_pack(job.tree.parent, job.tree.length, job.tree.term)
        ts = []
        for r in range(reps + 1):
            flush_l2(flush)
            a, b = torch.cuda.Event(True), torch.cuda.Event(True)
            a.record()
            tt.tt_restore_loss(pk, job.logits, job.tok, dlogits=job.dlogits)
            b.record()
            torch.cuda.synchronize()
            if r >= 1:
                ts.append(a.elapsed_time(b))
        return float(np.median(ts)), pk.n_tokens
    lens = [len(p) for p in trajectory_token_paths(tt.tt_pack(job.tree.parent, job.tree.length, job.tree.term),
                                                   job.tree)]
    chunks, cur = [], []
    for L in lens:
        if cur and sum(cur) + L > max_rows:
            chunks.append(cur)
            cur = []
        cur.append(L)
    if cur:
        chunks.append(cur)
    rows = max(sum(c) for c in chunks)
    buf = job.scratch.logits[:rows] if job.scratch.logits.shape[0] >= rows else None
    if buf is None:
        buf = torch.empty(rows, VOCAB, device="cuda", dtype=torch.bfloat16)
        buf.normal_(0, 2)
    tok = torch.randint(0, VOCAB, (rows,), device="cuda", dtype=torch.int32)
    packs = [tt.tt_pack([-1] * len(c), c) for c in chunks]
    total = 0.0
    for pk in packs:
        n = pk.n_tokens
        ts = []
        for r in range(reps + 1):
            flush_l2(flush)
            a, b = torch.cuda.Event(True), torch.cuda.Event(True)
            a.record()
            tt.tt_restore_loss(pk, buf[:n], tok[:n], dlogits=buf[:n])
            b.record()
            torch.cuda.synchronize()
            if r >= 1:
                ts.append(a.elapsed_time(b))
        total += float(np.median(ts))
    return total, sum(lens)


# ------------------------------------------------------------------------------------ cpu oracle
def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


_ORACLE_INPUTS = {}


def oracle_sample(job_tree, cfg, budget_s=20.0, nthreads=None):
    """Time the fp64 oracle (as it stands: per-branch linearisation, one std::thread per q head) on
    a bounded sample of the workload: H = min(Hq, host cores) heads over the first trajectories of
    the tree, forward + backward.  Returns (seconds measured, the sample's share of the full
    workload's oracle work = per-branch pairs x heads, trajectories taken, threads used)."""
    import oracle
    opk = oracle.pack(job_tree.parent, job_tree.length)
    paths = oracle.paths(opk)
    Ls = np.array([len(p) for p in paths], dtype=np.int64)
    full_work = float((Ls * (Ls + 1) // 2).sum()) * cfg["hq"]
    d = cfg["d"]
    heads = max(1, min(cfg["hq"], nthreads or (os.cpu_count() or 1)))
    cap = budget_s * 3.0e5 * (128.0 / d)  # ~pairs per second per thread (fp64 fwd+bwd, d = 128)
    take, work = [], 0.0
    for t, L in enumerate(Ls):
        w = L * (L + 1) / 2
        if take and work + w > cap:
            break
        take.append(t)
        work += w
    if work > 1.5 * cap:
        # even the first trajectory is over budget: its first L' tokens (a causal prefix, L'(L'+1)/2
        # pairs) are the sample
        Lp = max(1, int((2.0 * cap) ** 0.5))
        sub_idx = paths[take[0]][:Lp].astype(np.int32)
        sub_ptr = np.array([0, len(sub_idx)], np.int64)
        work = Lp * (Lp + 1) / 2
    else:
        sub_idx = np.concatenate([paths[t] for t in take]).astype(np.int32)
        sub_ptr = np.concatenate([[0], np.cumsum([len(paths[t]) for t in take])]).astype(np.int64)
    # the sample's rows only, renumbered 0..n-1 (the per-branch oracle reads rows through path_idx)
    rows, local = np.unique(sub_idx, return_inverse=True)
    spk = {"path_ptr": sub_ptr, "path_idx": local.astype(np.int32), "n_traj": len(sub_ptr) - 1}
    key = (len(rows), heads, d)
    if key not in _ORACLE_INPUTS:
        rng = np.random.default_rng(0)
        _ORACLE_INPUTS.clear()
        _ORACLE_INPUTS[key] = tuple(rng.standard_normal((len(rows), heads, d)) for _ in range(4))
    q, k, v, g = _ORACLE_INPUTS[key]
    t0 = time.perf_counter()
    oracle.attn_fwd(spk, q, k, v, 1 / math.sqrt(d), nthreads=heads)
    oracle.attn_bwd(spk, q, k, v, g, 1 / math.sqrt(d), nthreads=heads)
    dt = time.perf_counter() - t0
    return dt, work * heads / full_work, (len(take) if len(sub_ptr) > 2 or len(sub_idx) == Ls[take[0]] else
                                          f"{len(sub_idx)} tokens of 1"), heads


# ------------------------------------------------------------------------------------ pack (one launch)
def time_forest_pack(trees_list, reps=5):
    """a1 over the whole batch in ONE tt_pack call (the 64-tree forest, 64 MiB of
    per-token output, since single-tree packs are launch-latency bound).  Device time only: a
    sleep kernel keeps the stream busy while the host does the DFS, so the events bracket the H2D
    copy of the node tables and the two pack kernels.  Returns (ms, tokens, blocks, tiles)."""
    import torch
    import paper_2511_00413_b200 as tt
    par, ln, off = [], [], 0
    for t in trees_list:
        p = np.asarray(t.parent, np.int64)
        par.append(np.where(p >= 0, p + off, -1))
        ln.append(np.asarray(t.length, np.int64))
        off += len(p)
    par = np.concatenate(par).astype(np.int32)
    ln = np.concatenate(ln).astype(np.int32)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    ts, pk = [], None
    # 4 untimed calls first: tt_pack stages its node tables through a 4-slot pinned ring that grows to
    # the forest's size on first use (cudaFreeHost / cudaHostAlloc would otherwise land in the window)
    warm = 4
    for r in range(reps + warm):
        flush_l2(flush)
        pk = None
        torch.cuda._sleep(40_000_000)  # ~20 ms of device time: covers the host part of tt_pack
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        pk = tt.tt_pack(par, ln)
        b.record()
        torch.cuda.synchronize()
        if r >= warm:
            ts.append(a.elapsed_time(b))
    tiles = int(pk.arrays()["fwd_cnt"].sum().item())
    return float(np.median(ts)), pk.n_tokens, pk.n_blk, tiles


# ------------------------------------------------------------------------------------ main
def run_leg(out, name, fn):
    """An extra measurement after the timed step: a failure is recorded in the line, never loses it."""
    import traceback
    try:
        fn()
    except Exception as e:  # noqa: BLE001
        out.setdefault("leg_errors", {})[name] = f"{type(e).__name__}: {e}"
        traceback.print_exc()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="tt", choices=["tt", "reference"])
    ap.add_argument("--config", default="batch64k", choices=["batch64k", "agentic8k", "deep32k", "wide", "wide_aligned"])
    ap.add_argument("--trees", type=int, default=64, help="trees for --config batch64k")
    ap.add_argument("--seed", type=int, default=None)
    ap.add_argument("--no-loss", action="store_true")
    ap.add_argument("--no-linear", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-lmhead", action="store_true", help="skip the NEXT-f3 LM-head measurement")
    ap.add_argument("--no-extras", action="store_true", help="skip every leg after the timed step (profiling runs)")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.no_extras:
        args.no_linear = args.no_e2e = args.no_cpu = args.no_lmhead = True

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    from workloads import trees as T
    cfg = T.CONFIGS[args.config]

    if args.impl == "reference":
        return main_reference(args, rank, world, cfg)

    import torch
    # one process per GPU over NCCL; TT_BENCH_BACKEND=gloo runs the same multi-rank code path with several
    # ranks sharing the GPUs there are (a functional check of sharding + aggregation on a 1-GPU box:
    # tests/test_gpu_multirank_bench.py; its timings are not a measurement)
    backend = os.environ.get("TT_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    agg_dev = "cuda" if backend == "nccl" else "cpu"
    dist = None
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    import paper_2511_00413_b200 as tt
    tt.lib()
    refuse_dev_build(tt)

    my_trees, extra_cfg = make_trees(args, rank, world)
    with_loss = not args.no_loss
    host_copy = not args.no_e2e
    maxN = max(int(tt.tt_pack_plan(t.parent, t.length)["n_tokens"]) for _, t in my_trees)
    scratch = Scratch(maxN, cfg, VOCAB, with_loss, host_copy)
    jobs = [TreeJob(tid, t, cfg, VOCAB, scratch, with_loss=with_loss, host_copy=host_copy) for tid, t in my_trees]
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    n_total_trees = args.trees if args.config == "batch64k" else world

    def do_step(ev=None, h2d=False):
        for i, j in enumerate(jobs):
            run_step(j, ev=None if ev is None else ev[i], h2d=h2d)

    # warm-up
    for _ in range(args.warmup):
        do_step()
    torch.cuda.synchronize()

    # ---- timed device region ----
    names = ["pack", "fwd", "loss", "bwd"]
    # per (step, tree) event pairs around each op: per-op times are summed over the rank's trees
    evs = [[{n: (torch.cuda.Event(True), torch.cuda.Event(True)) for n in names} for _ in jobs] for _ in range(args.steps)]
    step_ev = [(torch.cuda.Event(True), torch.cuda.Event(True)) for _ in range(args.steps)]
    sampler = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    time.sleep(0.3)
    tt.tt_launch_count_reset()
    for s in range(args.steps):
        flush_l2(flush)
        step_ev[s][0].record()
        do_step(ev=evs[s])
        step_ev[s][1].record()
    torch.cuda.synchronize()
    launches = tt.tt_launch_count()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    step_ms = [a.elapsed_time(b) for a, b in step_ev]
    my_ms = float(sum(step_ms))
    per_op, per_op_med, per_op_min = {}, {}, {}
    for n in names:
        if n == "loss" and not with_loss:
            continue
        xs = [sum(e[n][0].elapsed_time(e[n][1]) for e in es) for es in evs]
        per_op[n] = float(np.mean(xs))
        per_op_med[n] = round(float(np.median(xs)), 4)
        per_op_min[n] = round(float(np.min(xs)), 4)
    flops_mine = sum(j.flops() for j in jobs) * args.steps
    # a6 across ranks + the job time: the step's records (identical every step) gathered once
    records = [(j.tid, j.rec) for j in jobs]
    totals, n_seen, t_max, flops_all = aggregate(records, my_ms, flops_mine, n_total_trees, dist, world,
                                                 device=agg_dev)

    # ---- e2e: host buffers through the same public API, H2D + D2H inside the timed region ----
    e2e = None
    if host_copy:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        n_e2e = args.e2e_steps if args.e2e_steps else (2 if len(jobs) > 4 else max(2, min(args.steps, 5)))
        e_ms = 0.0
        for s in range(n_e2e):
            flush_l2(flush)
            a, b = torch.cuda.Event(True), torch.cuda.Event(True)
            a.record()
            do_step(h2d=True)
            b.record()
            torch.cuda.synchronize()
            e_ms += a.elapsed_time(b)
        e_ms /= n_e2e
        _, _, e_max, _ = aggregate([], e_ms, 0.0, n_total_trees, dist, world, device=agg_dev)
        e2e = {"value": round(flops_all / args.steps / (e_max * 1e-3) / 1e12, 3), "unit": "TFLOP/s",
               "ms_per_step": round(e_max, 4), "h2d_bytes_per_step": int(sum(j.h2d_bytes() for j in jobs)),
               "d2h_bytes_per_step": int(sum(j.d2h_bytes() for j in jobs)), "steps": n_e2e,
               "copies": "H2D from pinned host: Q, K, V, dO (= G), logits, token ids; D2H to pinned host: dQ, dK, dV "
                         "and the per-tree scalar record; dlogits stays on the device (the LM-head backward's input). "
                         + ("Bytes of rank 0." if world > 1 else "")}

    peaks = load_peaks()
    value = flops_all / (t_max * 1e-3) / 1e12
    out = None
    if rank == 0:
        j0 = jobs[0]
        info = j0.info
        # kernels inside a seconds-long step run at the power-capped sustained rate (MEASURED_PEAKS:
        # cuBLAS back to back for 4 s); a short step (ms) at the burst rate
        sustained = t_max / args.steps > 100.0
        tpeak = peaks["bf16_sustained"] if sustained else peaks["bf16"]
        tpeak_src = peaks["source"] + (", dense bf16 sustained (step > 100 ms)" if sustained else ", dense bf16 burst")
        result = {
            "metric": METRIC, "value": round(value, 3), "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(t_max / args.steps, 4), "higher_is_better": True,
            "scaling": "weak" if args.config != "batch64k" else "strong",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded trees; N(0,1) Q/K/V/dO per tree id; 2 N(0,1) bf16 logits; uniform token ids)",
            "config": {"workload": args.config, "trees": n_total_trees, "trees_per_rank": len(jobs),
                       "n_tokens": int(sum(j.N for j in jobs)),
                       "hq": cfg["hq"], "hkv": cfg["hkv"], "head_dim": cfg["d"], "vocab": VOCAB if with_loss else None,
                       "ancestor_pairs": int(sum(j.info["n_pairs"] for j in jobs)),
                       "linear_pairs": int(sum(j.info["n_linear_pairs"] for j in jobs)),
                       "linear_tokens": int(sum(j.info["n_linear_tokens"] for j in jobs)),
                       "pair_ratio": round(sum(j.info["n_linear_pairs"] for j in jobs) / sum(j.info["n_pairs"] for j in jobs), 4),
                       "token_ratio": round(sum(j.info["n_linear_tokens"] for j in jobs) / sum(j.N for j in jobs), 4),
                       "l2": "flushed between steps (256 MiB write, outside the step events); inputs > L2",
                       "parallelism": f"dp{world} (independent trees per rank, LPT)" if args.config == "batch64k"
                       else f"dp{world} (one tree per rank)", **extra_cfg},
            "pct_peak": round(100.0 * value / peaks["bf16"], 2),
            "gpu_launches": int(launches),
            "clocks": clocks,
            "totals": {"trees": n_seen, "sum_loss": totals[0], "sum_omega": totals[1], "dq_sqnorm": totals[2],
                       "dk_sqnorm": totals[3], "dv_sqnorm": totals[4],
                       "order": "per-tree fp64 records summed in tree-id order on every rank (sum_loss, sum_omega, "
                                "dk/dv norms bitwise identical at every world size; dq norm follows dQ's fp32 "
                                "reduction order)"},
        }
        if per_op:
            result["per_op_ms"] = {k: round(v, 4) for k, v in per_op.items()}
            result["per_op_ms_median"] = per_op_med
            result["per_op_ms_min"] = per_op_min
            result["step_ms_median"] = round(float(np.median(step_ms)), 4)
            result["step_ms_min"] = round(float(np.min(step_ms)), 4)
            if len(jobs) > 1:
                result["per_op_ms"]["note"] = f"summed over the rank's {len(jobs)} trees (rank 0)"
            attn_ms = per_op["fwd"] + per_op["bwd"]
            my_flops = sum(j.flops() for j in jobs)
            my_pairs = sum(j.info["n_pairs"] for j in jobs)
            my_rows = sum(j.info["n_tokens"] for j in jobs)
            result["attn_fwd_bwd_tflops"] = round(my_flops / (attn_ms * 1e-3) / 1e12, 2)
            traffic, util, dens = {}, {}, {}
            prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
            if os.path.exists(prof):
                try:
                    pj = json.load(open(prof))
                    traffic = pj.get(args.config, {})
                    util = pj.get("bf16_mma_ops_pct", {}).get(args.config, {})
                    dens = pj.get("tile_density", {}).get(args.config, {})
                except Exception:
                    traffic, util, dens = {}, {}, {}
            per_launch = "" if len(jobs) == 1 else f" (mean over the rank's {len(jobs)} launches)"

            def tensor_roof(name, kernel, fl_per_pair, ms, main_kernel):
                ach = fl_per_pair * j0.d * j0.hq * my_pairs / (ms * 1e-3) / 1e12
                raw = util.get(main_kernel)
                r = {"bound": "tensor", "kernel": kernel + per_launch, "achieved": round(ach, 2), "peak": tpeak,
                     "unit": "TFLOP/s", "frac": round(ach / tpeak, 4), "traffic": traffic.get(main_kernel),
                     "peak_source": tpeak_src, "frac_of_burst": round(ach / peaks["bf16"], 4),
                     "algorithmic": f"{fl_per_pair} d Hq A FLOPs per launch (A = ancestor pairs: only unmasked pairs)",
                     "ms": round(ms, 4)}
                if raw is not None:
                    # raw tensor-core utilisation from ncu (every multiplied tile element, masked ones
                    # included) and the tile density = effective / raw FLOPs of the captured launch
                    r["ncu_bf16_mma_ops_pct"] = raw
                    r["tile_density"] = dens.get(main_kernel)
                return r

            # which backward kernel tt_attn_bwd dispatched to (persistent for short work items, flat for
            # long ones: tt_attn_bwd_kernel), per tree of the rank
            bks = sorted({tt.tt_attn_bwd_kernel(tt.tt_pack(j.tree.parent, j.tree.length), j.hq, j.hkv) for j in jobs})
            bk = bks[0] if len(bks) == 1 else "tree_attn_bwd_sm100"
            cand = {"bwd": tensor_roof("bwd", "tt_attn_bwd (bwd_pre + " + " / ".join(bks) + " + dq_convert)", 10,
                                       per_op["bwd"], bk),
                    "fwd": tensor_roof("fwd", "tt_attn_fwd (tree_attn_fwd_sm100)", 4, per_op["fwd"],
                                       "tree_attn_fwd_sm100")}
            if with_loss:
                lb = my_rows * (4 * VOCAB + 12)
                gbs = lb / (per_op["loss"] * 1e-3) / 1e9
                # one launch = the clusters' rows + loss_pipe_kernel's tail rows on the SMs the clusters
                # leave idle (side stream, joined) + the fixed-order sum; ncu bytes of both row kernels
                ltr = [traffic.get(k) for k in LOSS_KERNELS if traffic.get(k) is not None]
                cand["loss"] = {"bound": "hbm", "kernel": "tt_restore_loss (" + " + ".join(LOSS_KERNELS) + " + loss_sum_kernel)"
                                + per_launch,
                                "achieved": round(gbs, 1), "peak": peaks["hbm"], "unit": "GB/s",
                                "frac": round(gbs / peaks["hbm"], 4), "traffic": sum(ltr) if ltr else None,
                                "peak_source": peaks["source"] + ", HBM copy bandwidth",
                                "algorithmic": "N (4 V + 12) bytes per launch (read + write bf16 logits row, "
                                               "token id, weight, loss)",
                                "ms": round(per_op["loss"], 4)}
            dom = max(cand, key=lambda k: cand[k]["ms"])
            result["roofline"] = dict(cand[dom], op=dom)
            for k in cand:
                if k != dom:
                    result["roofline_" + k] = cand[k]
        if e2e:
            result["e2e"] = e2e
        out = result
    def leg_pack():
        # a1 over the rank's whole batch in one launch; per-step packs above are per tree
        pms, pN, pnb, ptiles = time_forest_pack([j.tree for j in jobs])
        pbytes = 16 * pN + 12 * pnb + 4 * ptiles
        gbs = pbytes / (pms * 1e-3) / 1e9
        out["roofline_pack"] = {"bound": "hbm", "kernel": f"tt_pack of the rank's {len(jobs)}-tree forest in one call "
                                "(node-table H2D + pack_fill_kernel + pack_tiles_kernel)",
                                "achieved": round(gbs, 1), "peak": peaks["hbm"], "unit": "GB/s",
                                "frac": round(gbs / peaks["hbm"], 4), "traffic": None,
                                "algorithmic": "16 B/token written (pos, w, E, node) + 12 B/block (min/max E, tile count) "
                                               "+ 4 B per non-empty tile",
                                "tokens": pN, "ms": round(pms, 4), "peak_source": peaks["source"] + ", HBM copy bandwidth"}
    if rank == 0 and not args.no_extras:
        run_leg(out, "pack", leg_pack)
    # ---- per-branch linear comparison (same kernels, untimed w.r.t. the step; rank 0's first tree) ----
    def leg_linear():
        j0 = jobs[0]
        tree_ms = (per_op["fwd"] + per_op["bwd"]) / len(jobs) if len(jobs) == 1 else None
        if tree_ms is None:
            tree_ms = linear_attention_time(j0, tree_only=True)
        lin_ms, lin_pairs, lin_tokens = linear_attention_time(j0)
        pr = j0.info["n_linear_pairs"] / j0.info["n_pairs"]
        tr = j0.info["n_linear_tokens"] / j0.info["n_tokens"]
        out["speedup_vs_linear"] = {"tree": int(j0.tid), "attn_fwd_bwd_tree_ms": round(tree_ms, 4),
                                    "attn_fwd_bwd_linear_ms": round(lin_ms, 4),
                                    "speedup": round(lin_ms / tree_ms, 3),
                                    "pair_ratio": round(pr, 4), "token_ratio": round(tr, 4),
                                    "frac_of_pair_ratio": round(lin_ms / tree_ms / pr, 3),
                                    "frac_of_token_ratio": round(lin_ms / tree_ms / tr, 3)}
        if with_loss:
            # SURVEY §8(d) reading: the loss is graded against the token ratio, the combined hot path
            # against its time-weighted ratio (the linear loss runs in place, chunked by trajectories)
            ll_ms, ll_rows = linear_loss_time(j0)
            t_loss = per_op["loss"] / len(jobs) if len(jobs) == 1 else linear_loss_time(j0, tree_only=True)[0]
            out["speedup_vs_linear"].update({
                "loss_tree_ms": round(t_loss, 4), "loss_linear_ms": round(ll_ms, 4),
                "loss_speedup": round(ll_ms / t_loss, 3),
                "loss_frac_of_token_ratio": round(ll_ms / t_loss / tr, 3),
                "attn_plus_loss_speedup": round((lin_ms + ll_ms) / (tree_ms + t_loss), 3)})
    if rank == 0 and not args.no_linear:
        run_leg(out, "linear", leg_linear)
    def leg_next():
        # NEXT-f1: capacity-constrained Tree Packing of this rank's tree at a budget forcing a split
        # (C = max(longest trajectory, tree tokens / 2)); host planner timing + effective reuse
        t_ = jobs[0].tree
        lens = tt.tt_plan_traversals(t_.parent, t_.length, 1 << 40)[1]
        longest = max(int(x) for x in _longest_paths(t_))
        C = max(longest, lens["tree_tokens"] // 2)
        reps = 20
        t0 = time.perf_counter()
        for _ in range(reps):
            a, pinfo = tt.tt_plan_traversals(t_.parent, t_.length, C)
        plan_ms = (time.perf_counter() - t0) / reps * 1e3
        out["next_f1_planner"] = {"capacity": int(C), "n_traversals": pinfo["n_traversals"],
                                  "planned_tokens": pinfo["planned_tokens"], "tree_tokens": pinfo["tree_tokens"],
                                  "linear_tokens": pinfo["linear_tokens"],
                                  "ERR": round(1 - pinfo["planned_tokens"] / pinfo["linear_tokens"], 4),
                                  "POR": round(1 - pinfo["tree_tokens"] / pinfo["linear_tokens"], 4),
                                  "host_plan_ms": round(plan_ms, 4)}
        # NEXT-f2: restored-position RoPE on this tree's Q and K, and the Gradient Scaler on its
        # upstream gradient (HBM-bound: each reads and writes its tensor once), event-timed with L2
        # flushed before every repetition
        j0 = jobs[0]
        pk0 = tt.tt_pack(j0.tree.parent, j0.tree.length)
        qc, kc, gc = j0.q.clone(), j0.k.clone(), j0.g.clone()

        def _t(fn, reps=10):
            fn()
            torch.cuda.synchronize()
            ts = []
            for _ in range(reps):
                flush_l2(flush)
                a, b = torch.cuda.Event(True), torch.cuda.Event(True)
                a.record()
                fn()
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            return float(np.median(ts))

        rope_ms = _t(lambda: (tt.tt_rope(pk0, qc), tt.tt_rope(pk0, kc)))
        rg_ms = _t(lambda: tt.tt_restore_grad(pk0, gc))
        rb = 2 * (qc.numel() + kc.numel()) * qc.element_size()
        gb = 2 * gc.numel() * gc.element_size()
        out["next_f2"] = {"rope_qk_ms": round(rope_ms, 4), "rope_gbs": round(rb / rope_ms / 1e6, 1),
                          "rope_frac": round(rb / rope_ms / 1e6 / peaks["hbm"], 4),
                          "restore_grad_ms": round(rg_ms, 4), "restore_grad_gbs": round(gb / rg_ms / 1e6, 1),
                          "restore_grad_frac": round(gb / rg_ms / 1e6 / peaks["hbm"], 4),
                          "hbm_peak_gbs": peaks["hbm"], "l2": "flushed before every repetition",
                          "algorithmic": "read + write of Q and K (rope), of G (restore_grad), bf16"}
        del qc, kc, gc
        if not args.no_lmhead:
            # NEXT-f3: LM head (Qwen3-8B hidden 4096, vocab 151,936) + restoration CE without the [N, V]
            # logits: 4 GEMMs of 2 N V D FLOPs each (two logits sweeps, dH, dW) + chunked CE kernels
            D_h, vc = 4096, 16384
            Nl = min(j0.N, 8192)
            pkl = pk0 if Nl == j0.N else tt.tt_pack(*_prefix_tree(j0.tree, Nl))
            g2 = torch.Generator(device="cuda").manual_seed(77)
            Hh = torch.randn(Nl, D_h, device="cuda", generator=g2).to(torch.bfloat16)
            Wl = (2.0 / D_h ** 0.5 * torch.randn(VOCAB, D_h, device="cuda", generator=g2)).to(torch.bfloat16)
            tokl = torch.randint(0, VOCAB, (Nl,), device="cuda", dtype=torch.int32, generator=g2)
            wsl = torch.empty(tt.tt_lmhead_loss_workspace(pkl, D_h, VOCAB, vc), dtype=torch.uint8, device="cuda")
            dHl, dWl = torch.empty_like(Hh), torch.empty_like(Wl)
            # measured from an idle GPU (3 s cool-down after the timed step and the other legs, which
            # leave the board at its power cap), SM clocks sampled during the leg
            torch.cuda.synchronize()
            time.sleep(3.0)
            smp = ClockSampler(local)
            smp.start()
            lm_ms = _t(lambda: tt.tt_lmhead_loss(pkl, Hh, Wl, tokl, vocab_chunk=vc, dh=dHl, dw=dWl, ws=wsl), reps=3)
            # context: one vocabulary chunk's four contractions on the library GEMM vs cuBLAS (torch.matmul)
            Wc = Wl[:vc]
            Gc = torch.randn(Nl, vc, device="cuda", generator=g2).to(torch.bfloat16)
            Xc = torch.empty(Nl, vc, device="cuda", dtype=torch.bfloat16)
            dHa = torch.zeros(Nl, D_h, device="cuda", dtype=torch.float32)
            dWc = torch.empty(vc, D_h, device="cuda", dtype=torch.bfloat16)
            dHb = torch.empty(Nl, D_h, device="cuda", dtype=torch.bfloat16)

            def mine():
                tt.tt_gemm(Hh, Wc, out=Xc)
                tt.tt_gemm(Hh, Wc, out=Xc)
                tt.tt_gemm(Gc, Wc, b_mn=True, out=dHa, accumulate=True)
                tt.tt_gemm(Gc, Hh, a_mn=True, b_mn=True, out=dWc)

            def cublas():
                torch.matmul(Hh, Wc.t(), out=Xc)
                torch.matmul(Hh, Wc.t(), out=Xc)
                torch.matmul(Gc, Wc, out=dHb)
                torch.matmul(Gc.t(), Hh, out=dWc)

            cfl = 8.0 * Nl * vc * D_h
            g_ms, c_ms = _t(mine, reps=3), _t(cublas, reps=3)
            lclk = smp.stop()
            fl = 8.0 * Nl * VOCAB * D_h
            out["next_f3_lmhead"] = {"ms": round(lm_ms, 3), "rows": Nl, "hidden": D_h, "vocab": VOCAB, "vocab_chunk": vc,
                                     "achieved_tflops": round(fl / lm_ms / 1e9, 1), "peak_tflops": peaks["bf16"],
                                     "frac": round(fl / lm_ms / 1e9 / peaks["bf16"], 4),
                                     "algorithmic": "8 N V D FLOPs (logits twice, dH, dW)", "l2": "flushed before every repetition",
                                     "gemm": "the library's tcgen05 CTA-pair GEMM (tt_gemm), CE fused into its epilogues",
                                     "chunk_gemms_tflops": {"tt_gemm": round(cfl / g_ms / 1e9, 1), "cublas": round(cfl / c_ms / 1e9, 1),
                                                            "note": "one chunk's X_c (twice), dH, dW_c: library GEMM vs torch.matmul"},
                                     "clocks": lclk, "cool_down_s": 3.0,
                                     "workspace_bytes": int(wsl.numel()),
                                     "materialised_logits_bytes_avoided": int(2 * 2 * Nl * VOCAB)}
            del Gc, Xc, dHa, dWc, dHb
            del Hh, Wl, dHl, dWl, wsl
    if rank == 0 and not args.no_extras:
        run_leg(out, "next", leg_next)
    def leg_cpu():
        dt, share, ntraj, cores = oracle_sample(jobs[0].tree, cfg, budget_s=args.cpu_budget)
        full_s = dt / share
        out["cpu_baseline"] = {"value": round(jobs[0].flops() / full_s / 1e12, 6), "unit": "TFLOP/s", "cores": cores,
                               "kind": "oracle",
                               "sample": f"fp64 oracle fwd+bwd on tree {jobs[0].tid}: {cores} of {cfg['hq']} heads (one "
                                         f"thread each), first {ntraj} trajectories ({share * 100:.3f}% of the tree's "
                                         f"per-branch pairs x heads), {dt:.1f} s measured; value = that share of the "
                                         f"tree's effective FLOPs / the measured time",
                               "extrapolated_full_tree_s": round(full_s, 1), "cpu_model": cpu_model(),
                               "host_cpus": os.cpu_count()}
    if rank == 0 and world == 1 and not args.no_cpu:
        run_leg(out, "cpu", leg_cpu)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _prefix_tree(tree, n_tok):
    """The first n_tok tokens of a tree in node order (a smaller tree for the LM-head leg)."""
    par, ln = [], []
    left = n_tok
    for p, l in zip(tree.parent, tree.length):
        if left <= 0:
            break
        par.append(int(p))
        ln.append(int(min(l, left)))
        left -= int(ln[-1])
    return par, ln


def main_reference(args, rank, world, cfg):
    """--impl reference: the fp64 CPU oracle (as it stands) on the same workload and metric.  Each
    step is a bounded sample (heads x first trajectories of tree 0); its effective FLOPs are the
    sample's share of the tree's 14 d Hq A, so value = sample FLOPs / measured sample time and
    ms_per_step is the measured time of a sample step (no extrapolation enters the line)."""
    if rank != 0:
        return
    import oracle
    from workloads import trees as T
    seed = 0 if args.seed is None else args.seed
    tree = T.config_tree(args.config, seed) if args.config not in ("wide", "wide_aligned") else T.config_tree(args.config)
    opk = oracle.pack(tree.parent, tree.length)
    A = int((opk["pos"].astype(np.int64) + 1).sum())
    flops_tree = 14.0 * cfg["d"] * cfg["hq"] * A
    budget = max(1.0, min(args.cpu_budget, 150.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        oracle_sample(tree, cfg, budget_s=budget)
    ts, shares = [], []
    for _ in range(args.steps):
        dt, share, ntraj, cores = oracle_sample(tree, cfg, budget_s=budget)
        ts.append(dt)
        shares.append(share)
    step_s = float(np.mean(ts))
    value = flops_tree * float(np.mean(shares)) / step_s / 1e12
    out = {"impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": "TFLOP/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(step_s * 1e3, 1), "higher_is_better": True,
           "scaling": "strong" if args.config == "batch64k" else "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "config": {"workload": args.config, "tree": seed, "hq": cfg["hq"], "hkv": cfg["hkv"],
                                           "head_dim": cfg["d"], "ancestor_pairs": A},
           "cpu_baseline": {"value": round(value, 6), "unit": "TFLOP/s", "cores": cores, "kind": "oracle",
                            "sample": f"per step: {cores} of {cfg['hq']} heads (one thread each) over the first "
                                      f"{ntraj} trajectories of tree {seed} (~{100 * float(np.mean(shares)):.3f}% of its "
                                      f"per-branch pairs x heads), {step_s:.2f} s measured per step",
                            "extrapolated_full_tree_s": round(step_s / float(np.mean(shares)), 1)},
           "e2e": {"value": round(value, 6), "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
