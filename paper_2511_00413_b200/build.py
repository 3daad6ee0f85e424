"""Build libtt.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension machinery).

    python -m paper_2511_00413_b200.build          # incremental
    python -m paper_2511_00413_b200.build --force

Every .cu under csrc/ is compiled with
    -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo
and linked into paper_2511_00413_b200/libtt.so (cudart static).  The .so travels to the GPU box
with the gpurun snapshot; it is git-ignored.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build")
SO = os.path.join(HERE, "libtt.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-Xptxas", "-warn-spills", "-I", os.path.join(ROOT, "include")]
# Development builds (--dev, or TT_DEV=1 in the environment): -DTT_DEV compiles in the environment
# A/B switches (ablations / variant sweeps, csrc/tt_internal.cuh dev_getenv) and, with
# TT_PROFILE_COUNTERS, per-role cycle counters; TT_EXTRA_NVCC_FLAGS adds compile-time variants.  The
# library reports it through tt_build_flags() and bench.py refuses to time it.
DEV_FLAGS = ["-DTT_DEV"]
if os.environ.get("TT_PROFILE_COUNTERS"):
    DEV_FLAGS += ["-DTT_PROFILE_COUNTERS"]
if os.environ.get("TT_EXTRA_NVCC_FLAGS"):
    DEV_FLAGS += os.environ["TT_EXTRA_NVCC_FLAGS"].split()


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _deps_mtime(src: str) -> float:
    hdrs = glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "tt.h")]
    return max([os.path.getmtime(src)] + [os.path.getmtime(h) for h in hdrs])


def build(force: bool = False, verbose: bool = False, dev: bool = False) -> str:
    dev = dev or bool(os.environ.get("TT_DEV"))
    flags = FLAGS + (DEV_FLAGS if dev else [])
    os.makedirs(OBJ, exist_ok=True)
    stamp = os.path.join(OBJ, "flags.txt")
    if not os.path.exists(stamp) or open(stamp).read() != " ".join(flags):
        force = True  # release <-> dev switch: rebuild every object
    
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    jobs = []
    for s in srcs:
        o = os.path.join(OBJ, os.path.basename(s)[:-3] + ".o")
        if force or not os.path.exists(o) or os.path.getmtime(o) < _deps_mtime(s):
            jobs.append((s, o))

    def comp(so):
        s, o = so
        cmd = [nvcc()] + ARCH + flags + ["-c", s, "-o", o]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {os.path.basename(s)}:\n{r.stderr}")
        return s, r.stderr

    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(8, len(jobs))) as ex:
            for s, err in ex.map(comp, jobs):
                if verbose and err.strip():
                    print(f"[{os.path.basename(s)}]\n{err}", file=sys.stderr)
    objs = [os.path.join(OBJ, os.path.basename(s)[:-3] + ".o") for s in srcs]
    if force or jobs or not os.path.exists(SO) or os.path.getmtime(SO) < max(os.path.getmtime(o) for o in objs):
        cuda_lib = os.path.join(os.path.dirname(os.path.dirname(os.path.realpath(nvcc()))), "lib64")
        cmd = [nvcc()] + ARCH + ["-shared", "-o", SO] + objs + ["-L" + cuda_lib, "-lcudart_static", "-ldl",
                                                               "-lrt", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    with open(stamp, "w") as f:
        f.write(" ".join(flags))
    return SO


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    ap.add_argument("--dev", action="store_true", help="development build (-DTT_DEV): env A/B switches compiled in")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose, dev=a.dev))
