"""bench.py's multi-rank path on real kernels.

The driver's 8-GPU step is not available to this build (one GPU per box), so this test runs
bench.py's own N > 1 code path — LPT sharding of config 5's trees, each rank's pack / fwd / loss /
bwd on its own trees, the record all_gather, the tree-id-ordered reduction and the max-over-ranks
time — as two ranks sharing the box's GPU, with gloo in place of NCCL for the two collectives
(TT_BENCH_BACKEND=gloo).  The reduced totals must equal the single-rank run's: sum loss, sum Omega,
|dK|^2 and |dV|^2 bitwise, |dQ|^2 to fp32-reduction-order rounding.
"""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _last_json(out):
    for ln in reversed(out.strip().splitlines()):
        ln = ln.strip()
        if ln.startswith("{"):
            return json.loads(ln)
    raise AssertionError("no JSON line in bench output:\n" + out[-2000:])


@pytest.mark.gpu
def test_bench_two_ranks_totals_match_one_rank():
    args = ["bench.py", "--trees", "4", "--steps", "1", "--warmup", "3", "--no-extras"]
    env = dict(os.environ, TT_BENCH_BACKEND="gloo")
    one = subprocess.run([sys.executable] + args, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert one.returncode == 0, one.stderr[-3000:]
    two = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(_free_port())] + args + ["--gpus", "2"],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    assert two.returncode == 0, two.stderr[-3000:]
    r1, r2 = _last_json(one.stdout), _last_json(two.stdout)
    assert r1["n_gpus"] == 1 and r2["n_gpus"] == 2
    assert r2["config"]["trees"] == 4 and 1 <= r2["config"]["trees_per_rank"] <= 3
    t1, t2 = r1["totals"], r2["totals"]
    assert t1["trees"] == t2["trees"] == 4
    for k in ("sum_loss", "sum_omega", "dk_sqnorm", "dv_sqnorm"):
        assert t1[k] == t2[k], (k, t1[k], t2[k])
    assert abs(t1["dq_sqnorm"] - t2["dq_sqnorm"]) <= 1e-6 * abs(t1["dq_sqnorm"])
