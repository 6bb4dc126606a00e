"""The measured serving loop pinned to the oracle (GPU, through the C-ABI).

bench.py times serving.ShardedEngine: two request shards on two CUDA
streams, each round ``duchess_score_active`` (K1 over the device-side
survivor list) + ``duchess_round`` (decide k, refill, advance k+1), device
probabilities (PRED_DEVICE). These tests run that exact loop with the
bench's workload recipe (bench.make_workload / make_probe) and the keyed
synthetic window source (activations keyed by (request, template,
position), regenerated on the CPU by oracle/activations.py), with every
snapshot taken on the shard streams (no host sync inside the loop), then:

* every request's RoundReports and outcome equal the oracle DuchessRun
  (oracle/port.py, pinned to the reference's golden vectors) fed the
  probability the device decided each survivor with through predictor=
  (reference seam orchestrator.py:319-327, :358-363);
* that probability equals the fp64 oracle probe of the regenerated window
  (mean over the L layers' probabilities at C3, combine=1) and sampled
  logits are within 1e-4*max(|ref|,1) (BASELINE.json north_star).
"""

import random

import numpy as np
import pytest
import torch

import bench
from oracle import activations as oact
from oracle import port
from tests.golden_util import port_report_tuple

pytestmark = pytest.mark.gpu


def _serve(cfg_name, R, pool, T, H, L, shards=2, seed=5):
    from paper_2509_24957_b200.engine import decode_round
    from paper_2509_24957_b200.probe import ProbeBank
    from paper_2509_24957_b200.scheduler import difficulty_queue
    from paper_2509_24957_b200.serving import ShardedEngine, keyed_fill
    cfg = dict(bench.CONFIGS[cfg_name], R=R, pool=pool, T=T, H=H, L=L)
    traces, knobs, seeds = bench.make_workload(cfg, seed=1000)
    w, b, g, beta = bench.make_probe(H, L)
    bank = ProbeBank.from_linear(w, b, g, beta)
    queue = difficulty_queue([t.difficulty for t in traces])
    srv = ShardedEngine(traces, knobs, seeds, bank, n_slots=R, shards=shards, queue=queue,
                        cycle=False, T=T, dtype=torch.bfloat16)
    fill = keyed_fill(seed)
    snaps = [[] for _ in range(shards)]
    pending = [None] * shards

    def fill_and_snap(k, eng, acts):
        fill(k, eng, acts)
        t = eng.t
        pending[k] = [t[n].clone() for n in ("row_mask", "row_req", "row_tmpl", "row_pos")]

    def after(k, eng):
        t = eng.t
        snaps[k].append(pending[k] + [t["step_pred"].clone(), srv.shards[k]["logit"].clone(),
                                      t["round_rec"].clone(), t["actions"].clone()])

    rounds = srv.run(max_rounds=2000, fill=fill_and_snap, after_round=after)
    torch.cuda.synchronize()
    C = knobs.max_branches
    seen, logits, reports = {}, {}, {}
    for k in range(shards):
        for mask, req, tm, pos, pred, lg, rec, act in snaps[k]:
            mask = mask.cpu().numpy().astype(bool)
            req, tm, pos = (x.cpu().numpy() for x in (req, tm, pos))
            pred, lg = pred.cpu().numpy(), lg.cpu().numpy()
            for row in np.nonzero(mask)[0]:
                key = (int(req[row]), int(tm[row]), int(pos[row]))
                assert key not in seen, "a (request, template, position) scored twice"
                seen[key] = float(pred[row])
                logits[key] = lg[row].copy()
            for p, rep in decode_round(rec.cpu().numpy(), act.cpu().numpy(), srv.Rs, C):
                reports.setdefault(p, []).append(rep)
    return srv, traces, knobs, seeds, (w, b, g, beta), seen, logits, reports, rounds


def _check(srv, traces, knobs, seeds, probe, seen, logits, reports, T, H, L, seed=5,
           n_logit_checks=48):
    from paper_2509_24957_b200 import _lib
    w, b, g, beta = probe
    cnt = srv.counters()
    assert int(cnt[_lib.CNT_AMBIGUOUS]) == 0
    assert int(cnt[_lib.CNT_BRANCH_STEPS]) == len(seen)
    outcomes = srv.outcomes()
    assert sorted(outcomes) == list(range(len(traces)))
    # scores: sampled windows regenerated on the CPU, fp64 probe
    keys = sorted(seen)
    rng = random.Random(0)
    for key in rng.sample(keys, min(n_logit_checks, len(keys))):
        ps = []
        for layer in range(L):
            win = oact.synth_window(seed, *key, layer, T, H, True)
            ref, pref = port.pooled_linear_probe(win, w[layer], float(b[layer]), g[layer],
                                                 beta[layer])
            assert abs(float(logits[key][layer]) - ref) <= 1e-4 * max(abs(ref), 1.0), key
            ps.append(pref)
        assert abs(seen[key] - sum(ps) / L) <= 1e-4, key
    # decisions: the oracle DuchessRun fed the device's probabilities
    for p, trace in enumerate(traces):
        index = {id(tp): j for j, tp in enumerate(trace.templates)}

        def predictor(tmpl, position, _rng, p=p, index=index):
            return seen[(p, index[id(tmpl)], position)]

        ref = port.DuchessRequest(trace, knobs, random.Random(seeds[p]), predictor=predictor)
        want = []
        while not ref.done:
            want.append(port_report_tuple(ref.step()))
        assert reports[p] == want, f"request {p}"
        o, got = ref.outcome, outcomes[p]
        assert (got["final"], got["reason"], got["tally"], got["tokens_decode"],
                got["tokens_probe"], got["rounds"]) == (
                    o.final, o.termination_reason, o.tally, o.tokens_decode, o.tokens_probe,
                    o.rounds), f"request {p}"


def test_bench_loop_c2_matches_oracle():
    """C2 as measured: 256 slots x 16 branches in 2 shards, T=32, H=4096 bf16,
    math-like knobs (c=16), 1024 requests served easiest-first (no cycling,
    so every request runs once and is checked)."""
    T, H, L = 32, 4096, 1
    out = _serve("c2", R=256, pool=1024, T=T, H=H, L=L)
    srv, traces, knobs, seeds, probe, seen, logits, reports, rounds = out
    assert len(seen) > 100_000 and rounds > 20
    _check(srv, traces, knobs, seeds, probe, seen, logits, reports, T, H, L)


def test_bench_loop_c3_four_layers_mean_combine_matches_oracle():
    """C3's shape with R scaled down: 64 slots x 32 branches in 2 shards,
    L=4 probe layers combined by the mean probability (round_kernel,
    combine=1), H=5120, T=32 bf16, 160 requests."""
    T, H, L = 32, 5120, 4
    out = _serve("c3", R=64, pool=160, T=T, H=H, L=L)
    srv, traces, knobs, seeds, probe, seen, logits, reports, rounds = out
    assert knobs.max_branches == 32 and len(seen) > 10_000
    _check(srv, traces, knobs, seeds, probe, seen, logits, reports, T, H, L)


def test_bench_loop_c3_t1_rows_kernel_matches_oracle():
    """C3-T1 (the paper's last-token probe, score_rows_kernel): L=4, T=1."""
    T, H, L = 1, 5120, 4
    out = _serve("c3t1", R=64, pool=160, T=T, H=H, L=L)
    _check(*out[:-1], T, H, L, n_logit_checks=200)
