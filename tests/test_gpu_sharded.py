"""The request-sharded multi-GPU inference path (distributed.run_sharded)
with two ranks, through the C-ABI.

Each rank is one process on the box's GPU (cuda:0 shared when only one is
visible); the host-side gathers run over gloo so two ranks can share a GPU
(on an 8-GPU node the same code runs one rank per GPU). Checked: the gathered
outcomes equal a single-rank run of the same workload, which equals the
oracle DuchessRun (oracle/port.py) fed the same probabilities — the per-
request seeds come from one master stream (request_seeds, as
simengine.py:191-193), so a request's decisions do not depend on its rank —
and the merged easiest-first order equals one global sort."""

import os
import random
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from oracle import activations as oact
from oracle import port

pytestmark = pytest.mark.gpu

H, T, L, SEED, MASTER = 512, 4, 2, 21, 77


def _workload():
    knobs = port.Knobs(max_branches=8, interval_tokens=16, early_term_threshold=0.7,
                       early_term_rounds=2, branch_out_temperature=0.8)
    params = port.GenParams(level_median_tokens=(120, 150, 200, 260, 300),
                            templates_per_request=24, probe_stride=16)
    traces = port.generate(params, 30, seed=12)
    rng = np.random.default_rng(3)
    w = rng.normal(0.0, 1.5 / np.sqrt(H), size=(L, H))
    g = rng.uniform(0.5, 1.5, size=(L, H))
    beta = rng.uniform(-0.1, 0.1, size=(L, H))
    return knobs, traces, (w, np.zeros(L), g, beta)


def _run(world_group_rank=None):
    from paper_2509_24957_b200.distributed import run_sharded
    from paper_2509_24957_b200.probe import ProbeBank
    knobs, traces, (w, b, g, beta) = _workload()
    bank = ProbeBank.from_linear(w, b, g, beta)
    return run_sharded(traces, knobs, MASTER, bank, n_slots=4, T=T, window_seed=SEED,
                       dtype=torch.bfloat16, shards=2, order="easiest")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port_, q):
    import torch.distributed as dist
    torch.cuda.set_device(rank % torch.cuda.device_count())
    # NCCL (the product's backend) when every rank has its own GPU; ranks sharing
    # one GPU use gloo (NCCL refuses two ranks on one device)
    backend = "nccl" if torch.cuda.device_count() >= world else "gloo"
    dist.init_process_group(backend, init_method=f"tcp://127.0.0.1:{port_}", rank=rank,
                            world_size=world)
    out, order = _run()
    if rank == 0:
        q.put(({p: (o["final"], o["reason"], o["tally"], o["tokens_decode"],
                    o["tokens_probe"], o["rounds"]) for p, o in out.items()}, order))
    dist.barrier()
    dist.destroy_process_group()


def _summary(out):
    return {p: (o["final"], o["reason"], o["tally"], o["tokens_decode"], o["tokens_probe"],
                o["rounds"]) for p, o in out.items()}


def test_two_rank_sharded_run_equals_one_rank_and_oracle():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_ = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port_, q)) for r in range(2)]
    for p in procs:
        p.start()
    two, order2 = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    one, order1 = _run()
    knobs, traces, _ = _workload()
    assert sorted(two) == list(range(len(traces)))
    assert two == _summary(one)
    # the merged order is one global easiest-first sort (level, order)
    want = sorted(range(len(traces)), key=lambda p: (traces[p].difficulty, p))
    assert order2 == want and order1 == want


def test_sharded_outcomes_equal_oracle_with_regenerated_probabilities():
    """Single rank: every request's outcome equals the oracle DuchessRun whose
    predictor scores the regenerated window of (request, template, position)
    with the fp64 probe (mean of the L layers' probabilities); probabilities
    within 1e-7 of a threshold are not expected at this size (checked)."""
    from paper_2509_24957_b200.distributed import request_seeds
    knobs, traces, (w, b, g, beta) = _workload()
    out, _ = _run()
    seeds, _ = request_seeds(len(traces), MASTER)
    for p, trace in enumerate(traces):
        index = {id(tp): j for j, tp in enumerate(trace.templates)}

        def predictor(tmpl, position, _rng, p=p, index=index):
            ps = []
            for layer in range(L):
                win = oact.synth_window(SEED, p, index[id(tmpl)], position, layer, T, H, True)
                ps.append(port.pooled_linear_probe(win, w[layer], 0.0, g[layer], beta[layer])[1])
            pr = sum(ps) / L
            assert abs(pr - knobs.early_term_threshold) > 1e-6
            return pr

        o = port.DuchessRequest(trace, knobs, random.Random(seeds[p]), predictor=predictor).run()
        got = out[p]
        assert (got["final"], got["reason"], got["tally"], got["tokens_decode"],
                got["rounds"]) == (o.final, o.termination_reason, o.tally, o.tokens_decode,
                                   o.rounds), f"request {p}"
