"""Randomised parity sweep: 40 random orchestration configurations (branch
slots 1-64, interval, threshold incl. disabled, streak length, temperature,
consensus / coverage fractions, token cap, probe cost, synthetic rho, template
counts) x a few requests each, with fewer device slots than requests (on-device
refill). The device engine (barrier-free duchess_round) must reproduce the CPU
oracle's RoundReports, outcomes and final branch states exactly; the oracle is
pinned to the reference's golden vectors (tests/test_oracle_golden.py)."""

import math
import random

import numpy as np
import pytest

from oracle import port
from tests.golden_util import STATUS, port_report_tuple

pytestmark = pytest.mark.gpu


def _config(rng):
    c = int(rng.choice([1, 2, 3, 5, 8, 12, 16, 24, 33, 48, 64]))
    knobs = port.Knobs(
        max_branches=c,
        interval_tokens=int(rng.choice([8, 16, 24, 40, 80])),
        early_term_threshold=float(rng.choice([0.5, 0.6, 0.7, 0.8, 0.9, math.inf])),
        early_term_rounds=int(rng.integers(1, 4)),
        branch_out_temperature=float(rng.choice([0.3, 0.5, 0.8, 1.0, 1.7])),
        consensus_frac=(cons := float(rng.choice([0.3, 0.5, 0.6, 1.0]))),
        coverage_frac=max(cons, float(rng.choice([0.5, 0.8, 1.0]))),
        token_cap=int(rng.choice([96, 256, 4096])),
        probe_cost_tokens=int(rng.choice([0, 10, 25])))
    params = port.GenParams(
        level_median_tokens=(180, 260, 340, 460, 640),
        templates_per_request=int(max(1, c + rng.integers(-c // 2, 2 * c + 3))),
        probe_stride=int(rng.choice([8, 16, 40])))
    return knobs, params, float(rng.choice([0.0, 0.5, 0.8, 1.0]))


@pytest.mark.parametrize("mode", ["split", "round"])
@pytest.mark.parametrize("seed", range(40))
def test_random_config_matches_oracle(seed, mode):
    """split: advance / decide launches (branch states inspected after each
    finish); round: the barrier-free duchess_round, whose same-launch refill
    reuses a finished slot at once, so only reports and outcomes are compared."""
    from paper_2509_24957_b200 import _lib
    from paper_2509_24957_b200.engine import BatchedDuchess
    rng = np.random.default_rng(1000 + seed)
    knobs, params, rho = _config(rng)
    traces = port.generate(params, 6, seed=seed)
    master = random.Random(seed)
    seeds = [master.getrandbits(64) for _ in traces]
    eng = BatchedDuchess(traces, knobs, seeds, n_slots=4, pred_source=_lib.PRED_TRACE, rho=rho)
    if mode == "round":
        eng.advance()
    reports, branches = {}, {}
    for _ in range(100000):
        if mode == "round":
            eng.round()
        else:
            eng.step()
        for p, rep in eng.round_reports():
            reports.setdefault(p, []).append(rep)
            if rep[6] and mode == "split":
                slot = int(np.nonzero(eng.t["slot_req"].cpu().numpy() == p)[0][0])
                snap = eng.branch_snapshot(slot)
                branches[p] = [(STATUS[int(s)], int(f), int(ob), int(td), int(st), int(n))
                               for s, f, ob, td, st, n in zip(
                                   snap["br_status"], snap["br_final"], snap["br_offset"],
                                   snap["br_decoded"], snap["br_streak"], snap["br_npred"])]
        if eng.all_done():
            break
    assert int(eng.counters()[_lib.CNT_AMBIGUOUS]) == 0
    outcomes = eng.outcomes()
    for p, tr in enumerate(traces):
        ref = port.DuchessRequest(tr, knobs, random.Random(seeds[p]), rho=rho)
        want = []
        while not ref.done:
            want.append(port_report_tuple(ref.step()))
        assert reports[p] == want, f"config {seed} request {p}"
        o = ref.outcome
        got = outcomes[p]
        assert (got["final"], got["reason"], got["tally"], got["tokens_decode"],
                got["tokens_probe"], got["rounds"]) == (
            o.final, o.termination_reason, o.tally, o.tokens_decode, o.tokens_probe, o.rounds)
        ans = eng.wl.answers[p]
        want_br = [(b.status, ans.index(b.final_answer) if b.final_answer is not None else -1,
                    b.offset_base, b.tokens_decoded, b.streak, len(b.prediction_history))
                   for b in ref.branches]
        if mode == "split":
            assert branches[p] == want_br, f"config {seed} request {p} branch states"
