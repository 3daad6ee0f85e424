"""bench.py's roofline_pack leg alone: one tt_pack of the 64-tree config-5 forest, device time (sleep
kernel covering the host DFS), plus ncu-free per-kernel event timing of the two pack kernels."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
from workloads import trees

ts = [trees.config_tree("batch64k", s) for s in range(64)]
for r in range(3):
    ms, N, nb, tiles = bench.time_forest_pack(ts)
    b = 16 * N + 12 * nb + 4 * tiles
    print(f"forest pack: {ms * 1e3:.1f} us for {N} tokens, {nb} blocks, {tiles} tiles -> {b / (ms * 1e-3) / 1e9:.0f} GB/s", flush=True)
