"""World-size-2 multi-process tests of the N>1 host logic on CPU (gloo):
request sharding + outcome gather, and the data-parallel gradient all-reduce."""

import os
import random
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import extensions as ext
from oracle import port


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _init(rank, world, port_):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port_}", rank=rank,
                           world_size=world)


def _sharded_requests(rank, world, port_, out_q):
    from paper_2509_24957_b200.distributed import gather_outcomes, request_seeds, shard_range
    _init(rank, world, port_)
    traces = port.generate(port.GenParams(templates_per_request=14), 10, seed=4)
    seeds, _ = request_seeds(len(traces), 11)
    knobs = port.Knobs(max_branches=6, interval_tokens=40, early_term_threshold=0.6)
    lo, hi = shard_range(len(traces), rank, world)
    local = {}
    for p in range(lo, hi):
        o = port.DuchessRequest(traces[p], knobs, random.Random(seeds[p]), rho=0.7).run()
        local[p] = (o.final, o.termination_reason, o.tokens_decode, o.tokens_probe, o.rounds)
    merged = gather_outcomes(local)
    if rank == 0:
        out_q.put(merged)
    dist.destroy_process_group()


def test_request_sharding_is_decision_invariant():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_ = _free_port()
    procs = [ctx.Process(target=_sharded_requests, args=(r, world, port_, q)) for r in range(world)]
    for p in procs:
        p.start()
    merged = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from paper_2509_24957_b200.distributed import request_seeds
    traces = port.generate(port.GenParams(templates_per_request=14), 10, seed=4)
    seeds, _ = request_seeds(len(traces), 11)
    knobs = port.Knobs(max_branches=6, interval_tokens=40, early_term_threshold=0.6)
    for p, tr in enumerate(traces):
        o = port.DuchessRequest(tr, knobs, random.Random(seeds[p]), rho=0.7).run()
        assert merged[p] == (o.final, o.termination_reason, o.tokens_decode, o.tokens_probe,
                             o.rounds)


def _dp_grad(rank, world, port_, out_q):
    from paper_2509_24957_b200.distributed import allreduce_sum, shard_range
    _init(rank, world, port_)
    rng = np.random.default_rng(0)
    N, H = 1001, 64
    X = rng.normal(size=(N, H)).astype(np.float32)
    y = (rng.random(N) < 0.5).astype(np.float32)
    w = rng.normal(size=H + 1) / 8
    lo, hi = shard_range(N, rank, world)
    part = ext.lr_grad_ref(X[lo:hi], y[lo:hi], w) * ((hi - lo) / N)
    t = torch.from_numpy(part.astype(np.float64))
    allreduce_sum(t)
    if rank == 0:
        out_q.put((t.numpy(), ext.lr_grad_ref(X, y, w)))
    dist.destroy_process_group()


def test_data_parallel_gradient_allreduce():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_ = _free_port()
    procs = [ctx.Process(target=_dp_grad, args=(r, world, port_, q)) for r in range(world)]
    for p in procs:
        p.start()
    got, want = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-14)


def test_shard_range_covers_everything():
    from paper_2509_24957_b200.distributed import shard_range
    for n in (0, 1, 7, 100, 1023):
        for world in (1, 2, 3, 8):
            spans = [shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1


def _difficulty_merge(rank, world, port_, out_q):
    from paper_2509_24957_b200.distributed import merge_difficulty_order, shard_range
    from paper_2509_24957_b200.scheduler import pack_keys
    _init(rank, world, port_)
    rng = np.random.default_rng(3)
    n = 500
    levels = rng.integers(1, 6, n)
    arrivals = rng.integers(0, 10 ** 6, n)
    keys = pack_keys(levels, arrivals, range(n))
    lo, hi = shard_range(n, rank, world)
    local = sorted(int(k) for k in keys[lo:hi])     # each rank's device sort (ordering only)
    merged = merge_difficulty_order(local)
    if rank == 0:
        out_q.put((merged, sorted(int(k) for k in keys)))
    dist.destroy_process_group()


def test_difficulty_order_merges_across_ranks():
    """per-rank sorted segments, all-gathered and k-way merged on
    the host, equal one global sort of the (level, arrival, order) keys."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_ = _free_port()
    procs = [ctx.Process(target=_difficulty_merge, args=(r, 2, port_, q)) for r in range(2)]
    for p in procs:
        p.start()
    merged, want = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
    assert merged == want
