"""Multi-GPU plumbing (one process per GPU, torch.distributed).

Requests are independent (reference SPEC.md:295: no shared mutable state
between requests; per-request RNG streams seeded in workload order,
simengine.py:191-193), so the inference path shards contiguous request ranges
across ranks with no collective; outcomes are gathered on the host at the end.
The only data-path collective is the probe-training gradient all-reduce
(train.py).
"""

from __future__ import annotations

import random


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [lo, hi) share of n items for `rank` (first ranks take the remainder)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def request_seeds(n: int, master_seed: int) -> tuple[list[int], list[int]]:
    """Per-request policy and difficulty-prediction seeds, drawn from one
    master stream in workload order exactly as simengine.py:191-193, so a
    request's stream does not depend on which rank serves it."""
    master = random.Random(master_seed)
    policy = [master.getrandbits(64) for _ in range(n)]
    predict = [master.getrandbits(64) for _ in range(n)]
    return policy, predict


def allreduce_sum(t, group=None):
    """In-place SUM all-reduce across the group (NCCL for CUDA tensors, gloo
    for CPU); a no-op without an initialised multi-rank process group."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def gather_outcomes(local: dict, group=None) -> dict:
    """Merge {pool index: outcome} dicts from every rank (host-side gather)."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return dict(local)
    parts = [None] * dist.get_world_size(group)
    dist.all_gather_object(parts, local, group=group)
    merged = {}
    for p in parts:
        merged.update(p)
    return merged


def merge_difficulty_order(local_sorted_keys, group=None) -> list:
    """Global easiest-first order across ranks: each rank
    sorts its own segment of 64-bit (level, arrival, order) keys on its GPU
    (scheduler.device_sort); the sorted runs are all-gathered (8 B per
    request) and k-way merged on the host. Keys are unique, so the merge equals
    one global sort (scheduler.py:60-96 pops over the union snapshot)."""
    import heapq

    import torch.distributed as dist
    local = [int(k) for k in local_sorted_keys]
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return local
    runs = [None] * dist.get_world_size(group)
    dist.all_gather_object(runs, local, group=group)
    return list(heapq.merge(*runs))
