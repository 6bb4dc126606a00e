"""Multi-GPU plumbing (one process per GPU, torch.distributed).

Requests are independent (reference SPEC.md:295: no shared mutable state
between requests; per-request RNG streams seeded in workload order,
simengine.py:191-193), so the inference path shards contiguous request ranges
across ranks with no collective (``run_sharded``): every rank packs the pool,
derives every request's seed from the one master stream, serves only its
``shard_range`` share through ``serving.ShardedEngine``, and the outcomes
(a few hundred bytes per request) are gathered on the host at the end. The
only data-path collective is the probe-training gradient all-reduce
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


def run_sharded(traces, config, master_seed: int, bank, *, n_slots: int, T: int,
                window_seed: int, dtype=None, shards: int = 2, order: str = "easiest",
                group=None, device=None, max_rounds: int = 100000):
    """Serve a workload across the ranks of `group` (one GPU per rank).

    traces: the whole pool (every rank packs it, so pool indices and the
    activation keys are global). Seeds: request_seeds(len(traces),
    master_seed)[0], i.e. random.Random(seed) per request drawn from one master
    stream in workload order (simengine.py:191-193), so a request's decisions
    do not depend on the rank serving it. This rank serves
    shard_range(len(traces), rank, world) with `n_slots` request slots split
    over `shards` CUDA streams; activations come from the keyed synthetic
    window source (serving.keyed_fill(window_seed)). order: "easiest" (each
    rank device-sorts its segment by (level, order), scheduler.py:76-90) or
    "fcfs" (pool order).

    Returns (outcomes, order): {pool index: outcome dict} for the whole pool
    (gathered from every rank) and the global easiest-first service order
    (per-rank device-sorted runs k-way merged, merge_difficulty_order).
    """
    import torch
    import torch.distributed as dist

    from .scheduler import device_sort, pack_keys
    from .serving import ShardedEngine, keyed_fill

    dtype = torch.bfloat16 if dtype is None else dtype
    multi = dist.is_available() and dist.is_initialized()
    rank = dist.get_rank(group) if multi else 0
    world = dist.get_world_size(group) if multi else 1
    device = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    P = len(traces)
    seeds, _ = request_seeds(P, master_seed)
    lo, hi = shard_range(P, rank, world)
    if order == "easiest":
        lv = [1 if traces[p].difficulty is None else traces[p].difficulty for p in range(lo, hi)]
        keys = pack_keys(lv, [0] * (hi - lo), range(lo, hi))
        local = [lo + j for j in device_sort(keys, device=device)]
        local_keys = [int(keys[p - lo]) for p in local]
    elif order == "fcfs":
        local, local_keys = list(range(lo, hi)), list(range(lo, hi))
    else:
        raise ValueError(f"unknown order {order!r}")
    outcomes = {}
    if hi > lo:
        shards = max(1, min(shards, n_slots))
        while n_slots % shards:
            shards -= 1
        eng = ShardedEngine(traces, config, seeds, bank, n_slots=n_slots, shards=shards,
                            queue=local, cycle=False, T=T, dtype=dtype, device=device)
        eng.run(max_rounds=max_rounds, fill=keyed_fill(window_seed))
        outcomes = eng.outcomes()
        if set(outcomes) != set(range(lo, hi)):
            raise RuntimeError("rank finished a different request set than it was given")
    merged = gather_outcomes(outcomes, group)
    if order == "easiest":
        pos = {k: p for k, p in zip(local_keys, local)}
        all_pos = gather_outcomes(pos, group)
        global_order = [all_pos[k] for k in merge_difficulty_order(local_keys, group)]
    else:
        global_order = list(range(P))
    return merged, global_order
