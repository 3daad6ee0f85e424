"""Multi-GPU sharding of independent trees.

Trees are independent units: the hot path has no exchange.  Work is partitioned across ranks by
greedy LPT on the per-tree attention work (ancestor pairs A, from tt_pack_plan), descending, ties
by tree id — deterministic.  After each step every rank contributes fixed-size per-tree records
[tree id, sum loss, sum Omega, |dQ|^2, |dK|^2, |dV|^2]; one all_gather_into_tensor (NCCL over
NVLink on the box, gloo in the CPU tests) collects them and every rank sums them in tree-id order,
so the totals are bitwise identical at every world size.
"""
from __future__ import annotations

import math
from typing import List, Sequence, Tuple

REC = 6  # tree id + 5 scalars


def lpt_partition(work: Sequence[int], world: int) -> Tuple[List[List[int]], float]:
    """Greedy longest-processing-time partition.  Returns (tree ids per rank, imbalance =
    max rank load / mean rank load)."""
    order = sorted(range(len(work)), key=lambda i: (-work[i], i))
    load = [0] * world
    assign: List[List[int]] = [[] for _ in range(world)]
    for i in order:
        r = min(range(world), key=lambda x: (load[x], x))
        assign[r].append(i)
        load[r] += work[i]
    mean = sum(load) / world if world else 0.0
    return [sorted(a) for a in assign], (max(load) / mean if mean else 1.0)


def slot_size(n_trees: int, world: int) -> int:
    # LPT may give one rank more than ceil(n / world) trees (many light trees vs a few heavy ones),
    # so every slot holds all n_trees records (a few KB)
    return n_trees * REC


def pack_records(records, n_trees: int, world: int, device=None):
    """records: list of (tree_id, [5 floats]) of this rank -> fixed-size fp64 slot (-1 padded)."""
    import torch
    out = torch.full((slot_size(n_trees, world),), -1.0, dtype=torch.float64, device=device)
    for k, (tid, vals) in enumerate(records):
        out[k * REC] = float(tid)
        if isinstance(vals, torch.Tensor):
            out[k * REC + 1:(k + 1) * REC].copy_(vals)
        else:
            out[k * REC + 1:(k + 1) * REC] = torch.as_tensor(vals, dtype=torch.float64, device=device)
    return out


def gather_records(slot, dist_mod, world: int):
    """One all_gather_into_tensor of every rank's slot."""
    import torch
    out = torch.empty(slot.numel() * world, dtype=slot.dtype, device=slot.device)
    dist_mod.all_gather_into_tensor(out, slot)
    return out


def reduce_records(gathered) -> Tuple[List[float], int]:
    """Sum the 5 scalars over all trees in tree-id order (deterministic).  Returns (totals, n)."""
    import torch
    g = gathered.detach().to("cpu", torch.float64).reshape(-1, REC)
    rows = [r for r in g.tolist() if r[0] >= 0]
    rows.sort(key=lambda r: r[0])
    tot = [0.0] * (REC - 1)
    for r in rows:
        for k in range(REC - 1):
            tot[k] += r[k + 1]
    return tot, len(rows)
