"""Multi-rank host logic on CPU (gloo, world size 2): LPT partition of independent trees and the
deterministic all_gather + tree-id-ordered reduction of per-tree scalars."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_00413_b200 import sharding


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _fake_record(tid):
    g = torch.Generator().manual_seed(1000 + tid)
    return [float(x) for x in torch.rand(5, generator=g, dtype=torch.float64) * 10 ** (tid % 7)]


def _worker(rank, world, port, n_trees, work, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    assign, _ = sharding.lpt_partition(work, world)
    recs = [(t, _fake_record(t)) for t in assign[rank]]
    slot = sharding.pack_records(recs, n_trees, world)
    g = sharding.gather_records(slot, dist, world)
    tot, n = sharding.reduce_records(g)
    out_q.put((rank, tot, n, assign[rank]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_gather_and_reduce(world):
    n_trees = 11
    work = [int(x) for x in torch.randint(1, 10 ** 6, (n_trees,), generator=torch.Generator().manual_seed(3))]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_trees, work, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # every rank sees all trees and identical totals
    ref = [0.0] * 5
    for t in range(n_trees):
        for k, v in enumerate(_fake_record(t)):
            ref[k] += v
    assigned = sorted(t for r in res for t in r[3])
    assert assigned == list(range(n_trees))
    for rank, tot, n, _ in res:
        assert n == n_trees
        assert tot == ref  # bitwise: same summation order as the single-process reference


def test_lpt_partition_properties():
    work = [5, 9, 1, 9, 3, 7, 2]
    assign, imb = sharding.lpt_partition(work, 3)
    assert sorted(sum(assign, [])) == list(range(7))
    loads = [sum(work[i] for i in a) for a in assign]
    assert max(loads) - min(loads) <= max(work)
    assert imb >= 1.0
    # deterministic and world-size-1 identity
    assert sharding.lpt_partition(work, 3) == (assign, imb)
    assert sharding.lpt_partition(work, 1)[0] == [list(range(7))]


def test_reduce_is_world_size_invariant():
    n_trees = 9
    recs = {t: _fake_record(t) for t in range(n_trees)}
    totals = []
    for world in (1, 2, 4):
        assign, _ = sharding.lpt_partition(list(range(1, n_trees + 1)), world)
        slots = [sharding.pack_records([(t, recs[t]) for t in assign[r]], n_trees, world) for r in range(world)]
        totals.append(sharding.reduce_records(torch.cat(slots))[0])
    assert totals[0] == totals[1] == totals[2]


def test_unequal_lpt_counts_fit_the_record_slot():
    """Three heavy trees and many light ones: LPT gives the fourth rank all the light trees, more than
    ceil(n / world); every rank's records must still fit its all_gather slot."""
    work = [1000, 1000, 1000] + [1] * 9
    world = 4
    assign, _ = sharding.lpt_partition(work, world)
    assert max(len(a) for a in assign) > -(-len(work) // world)
    recs = {t: _fake_record(t) for t in range(len(work))}
    slots = [sharding.pack_records([(t, recs[t]) for t in assign[r]], len(work), world) for r in range(world)]
    tot, n = sharding.reduce_records(torch.cat(slots))
    assert n == len(work)
    ref = [0.0] * 5
    for t in range(len(work)):
        for k, v in enumerate(recs[t]):
            ref[k] += v
    assert tot == ref


def _bench_worker(rank, world, port, n_trees, work, out_q):
    """bench.py's own step aggregation (bench.aggregate) on gloo: LPT partition, fixed-size record
    all_gather, tree-id-ordered reduction, max-over-ranks time and summed FLOPs."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    assign, _ = sharding.lpt_partition(work, world)
    recs = [(t, torch.tensor(_fake_record(t), dtype=torch.float64)) for t in assign[rank]]
    my_ms = 10.0 + rank
    my_flops = float(sum(work[t] for t in assign[rank]))
    tot, n, t_max, flops = bench.aggregate(recs, my_ms, my_flops, n_trees, dist, world, device=None)
    out_q.put((world, rank, tot, n, t_max, flops))
    dist.barrier()
    dist.destroy_process_group()


def test_bench_aggregate_world_sizes_bitwise():
    """the totals bench.py prints are bitwise identical at world sizes 1, 2 and 4 (the
    same per-tree records, gathered and summed in tree-id order), the job time is the max over
    ranks and the FLOPs are summed over ranks."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    n_trees = 13
    work = [int(x) for x in torch.randint(1, 10 ** 6, (n_trees,), generator=torch.Generator().manual_seed(5))]
    recs1 = [(t, torch.tensor(_fake_record(t), dtype=torch.float64)) for t in range(n_trees)]
    ref, n1, t1, f1 = bench.aggregate(recs1, 10.0, float(sum(work)), n_trees)
    assert n1 == n_trees and t1 == 10.0 and f1 == float(sum(work))
    ctx = mp.get_context("spawn")
    for world in (2, 4):
        q = ctx.Queue()
        port = _free_port()
        procs = [ctx.Process(target=_bench_worker, args=(r, world, port, n_trees, work, q)) for r in range(world)]
        for p in procs:
            p.start()
        res = [q.get(timeout=180) for _ in range(world)]
        for p in procs:
            p.join(timeout=60)
            assert p.exitcode == 0
        for w, rank, tot, n, t_max, flops in res:
            assert n == n_trees
            assert tot == ref, (world, rank)          # bitwise
            assert t_max == 10.0 + world - 1          # max over ranks
            assert flops == float(sum(work))
