"""GPU check behind bench.py's "totals identical at every world size": a tree's
per-tree record [sum loss, sum Omega, |dQ|^2, |dK|^2, |dV|^2] depends only on the tree, not on
which other trees the rank processed before it or in what order (as LPT assigns them differently
at every world size).  sum loss, sum Omega, |dK|^2 and |dV|^2 are bitwise equal; |dQ|^2 follows the
fp32 reduction order of dQ (within 1e-6 relative)."""
import os
import sys

import pytest

pytestmark = pytest.mark.gpu
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def test_records_independent_of_rank_assignment():
    import torch
    import bench
    import paper_2511_00413_b200 as tt
    from workloads import trees
    tt.lib()
    cfg = {"hq": 4, "hkv": 2, "d": 128}
    V = 4096
    ts = {tid: trees.gen_agentic(3000 + 500 * tid, root_len=400, seed=tid) for tid in range(3)}
    maxN = max(int(t.length.sum()) for t in ts.values())
    scratch = bench.Scratch(maxN, cfg, V, with_loss=True, host_copy=False)
    recs = []
    for order in ([0, 1, 2], [2, 0, 1], [1, 2]):
        jobs = [bench.TreeJob(t, ts[t], cfg, V, scratch) for t in order]
        for j in jobs:
            bench.run_step(j)
        torch.cuda.synchronize()
        recs.append({j.tid: j.rec.cpu().clone() for j in jobs})
    for tid in (0, 1, 2):
        seen = [r[tid] for r in recs if tid in r]
        for r in seen[1:]:
            assert torch.equal(r[[0, 1, 3, 4]], seen[0][[0, 1, 3, 4]]), tid
            assert abs(float(r[2]) - float(seen[0][2])) <= 1e-6 * float(seen[0][2])
    tot = [bench.aggregate([(t, recs[k][t]) for t in sorted(recs[k])], 1.0, 1.0, 3)[0] for k in (0, 1)]
    assert tot[0][0] == tot[1][0] and tot[0][1] == tot[1][1] and tot[0][3:] == tot[1][3:]
