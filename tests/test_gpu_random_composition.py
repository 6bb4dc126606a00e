"""Randomised K1 -> K2 composition: random orchestration configurations with
the probabilities produced by the probe scorer on windows keyed by
(request, template, position) — T = 1 (one warp per window) and T = 4 (CTA
kernel) — must drive the device decisions exactly as the oracle DuchessRun
decides when fed the same probabilities through predictor= (the reference
seam, orchestrator.py:319-327, :358-363)."""

import random

import numpy as np
import pytest
import torch

from oracle import port
from tests.golden_util import port_report_tuple
from tests.test_gpu_random_configs import _config

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", range(16))
def test_random_composition_matches_oracle(seed):
    from paper_2509_24957_b200 import _lib
    from paper_2509_24957_b200.engine import BatchedDuchess
    from paper_2509_24957_b200.probe import ProbeBank, Scorer, fill_windows
    rng = np.random.default_rng(5000 + seed)
    knobs, params, _rho = _config(rng)
    T = 1 if seed % 2 == 0 else 4
    H, L, R = 512, 1, 3
    traces = port.generate(params, 5, seed=100 + seed)
    master = random.Random(seed)
    seeds = [master.getrandbits(64) for _ in traces]
    w = rng.normal(0.0, 1.5 / np.sqrt(H), size=(1, H))
    g = rng.uniform(0.5, 1.5, size=(1, H))
    beta = rng.uniform(-0.1, 0.1, size=(1, H))
    # a bias that centres the logits near the decision thresholds
    bank = ProbeBank.from_linear(w, [float(rng.uniform(-0.5, 1.5))], g, beta)
    eng = BatchedDuchess(traces, knobs, seeds, n_slots=R, pred_source=_lib.PRED_DEVICE)
    C = knobs.max_branches
    acts = torch.zeros((R * C, L, T, H), dtype=torch.bfloat16, device="cuda")
    scorer = Scorer(bank, R * C * L)
    logit = torch.zeros((R * C, L), device="cuda")
    seen = {}

    def score(e):
        t = e.t
        fill_windows(acts, seed, t["row_req"], t["row_tmpl"], t["row_pos"], t["row_mask"])
        scorer(acts, logit, e.probs.view(R * C, L), row_mask=t["row_mask"])

    reports = {}
    for _ in range(100000):
        eng.step(score_fn=score)
        t = eng.t
        mask = t["row_mask"].cpu().numpy().astype(bool)
        keys = zip(t["row_req"].cpu().numpy(), t["row_tmpl"].cpu().numpy(),
                   t["row_pos"].cpu().numpy())
        pr = eng.probs.cpu().numpy()
        for row, (rq, tm, ps) in enumerate(keys):
            if mask[row]:
                seen[(int(rq), int(tm), int(ps))] = float(pr[row])
        for p, rep in eng.round_reports():
            reports.setdefault(p, []).append(rep)
        if eng.all_done():
            break
    assert int(eng.counters()[_lib.CNT_AMBIGUOUS]) == 0
    outcomes = eng.outcomes()
    for p, trace in enumerate(traces):
        index = {id(tp): j for j, tp in enumerate(trace.templates)}

        def predictor(tmpl, position, _rng, p=p, index=index):
            return seen[(p, index[id(tmpl)], position)]

        ref = port.DuchessRequest(trace, knobs, random.Random(seeds[p]), predictor=predictor)
        want = []
        while not ref.done:
            want.append(port_report_tuple(ref.step()))
        assert reports[p] == want, f"config {seed} request {p}"
        o = ref.outcome
        assert (outcomes[p]["final"], outcomes[p]["reason"], outcomes[p]["tally"]) == (
            o.final, o.termination_reason, o.tally)
