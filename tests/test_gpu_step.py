"""Fused round kernel (duchess_step: K1 scoring + decide + advance in one
persistent launch) on the GPU, through the C-ABI.

Parity: every request's RoundReports, outcome and tally equal the oracle
DuchessRun (oracle/port.py, pinned to the reference's golden vectors) fed the
same probabilities through predictor= (the reference seam,
orchestrator.py:319-327, :358-363); logits within 1e-4*max(|ref|,1) of the
fp64 oracle probe on the regenerated windows (tolerance from BASELINE.json
north_star)."""

import random

import numpy as np
import pytest
import torch

from oracle import activations as oact
from oracle import port
from tests.golden_util import port_report_tuple

pytestmark = pytest.mark.gpu


def _setup(n_req, c, temperature, templates=64):
    knobs = port.Knobs(max_branches=c, interval_tokens=16, early_term_threshold=0.70,
                       early_term_rounds=2, branch_out_temperature=temperature,
                       consensus_frac=0.6, coverage_frac=0.8)
    params = port.GenParams(level_median_tokens=(180, 220, 260, 300, 350),
                            level_correct_prob=(0.92, 0.88, 0.84, 0.80, 0.75),
                            templates_per_request=templates, probe_stride=16)
    traces = port.generate(params, n_req, seed=7)
    master = random.Random(11)
    seeds = [master.getrandbits(64) for _ in traces]
    return knobs, traces, seeds


def _probe(H, L):
    rng = np.random.default_rng(0)
    w = rng.normal(0.0, 1.5 / np.sqrt(H), size=(L, H))
    g = rng.uniform(0.5, 1.5, size=(L, H))
    beta = rng.uniform(-0.1, 0.1, size=(L, H))
    return w, g, beta


@pytest.mark.parametrize("dtype,T,H,L,c,R,temperature", [
    (torch.float32, 1, 4096, 1, 8, 8, 1.0),        # C1 shape
    (torch.bfloat16, 32, 4096, 1, 16, 12, 0.8),    # C2 shape, few slots (refills)
    (torch.bfloat16, 8, 1024, 2, 8, 5, 1.0),       # two probe layers, mean combine
    (torch.float32, 3, 520, 1, 4, 3, 0.5),         # odd T, H not a power of two
])
def test_fused_step_matches_oracle(dtype, T, H, L, c, R, temperature):
    from paper_2509_24957_b200 import _lib
    from paper_2509_24957_b200.engine import BatchedDuchess
    from paper_2509_24957_b200.probe import ProbeBank, fill_windows
    seed = 3
    knobs, traces, seeds = _setup(24, c, temperature)
    w, g, beta = _probe(H, L)
    bank = ProbeBank.from_linear(w, np.zeros(L), g, beta)
    eng = BatchedDuchess(traces, knobs, seeds, n_slots=R, pred_source=_lib.PRED_DEVICE,
                         n_layers=L, combine=1 if L > 1 else 0)
    C = knobs.max_branches
    acts = torch.zeros((R * C, L, T, H), dtype=dtype, device="cuda")
    logit = torch.zeros(R * C * L, device="cuda")
    seen, reports = {}, {}
    checked = 0
    eng.begin_fused()
    for _ in range(5000):
        t = eng.t
        fill_windows(acts, seed, t["row_req"], t["row_tmpl"], t["row_pos"], t["row_mask"])
        mask = t["row_mask"].cpu().numpy().astype(bool)
        req, tm, pos = (t[k].cpu().numpy() for k in ("row_req", "row_tmpl", "row_pos"))
        rows, n = eng.fused_rows()
        assert sorted(rows.cpu().tolist()) == list(np.nonzero(mask)[0])
        eng.step_fused(acts, bank, logit)
        # the prediction each survivor was decided with (eng.probs already
        # holds the next round's unscored sentinels)
        pr = eng.t["step_pred"].cpu().numpy()
        lg = logit.view(R * C, L).cpu().numpy()
        for row in np.nonzero(mask)[0]:
            key = (int(req[row]), int(tm[row]), int(pos[row]))
            seen[key] = float(pr[row])
            if checked < 120 and row % 3 == 0:
                ps = []
                for l in range(L):
                    win = oact.synth_window(seed, *key, l, T, H, dtype == torch.bfloat16)
                    ref, pref = port.pooled_linear_probe(win, w[l], 0.0, g[l], beta[l])
                    assert abs(float(lg[row, l]) - ref) <= 1e-4 * max(abs(ref), 1.0)
                    ps.append(pref)
                assert abs(seen[key] - sum(ps) / L) <= 1e-4
                checked += 1
        for p, rep in eng.round_reports():
            reports.setdefault(p, []).append(rep)
        if eng.all_done():
            break
    assert eng.all_done()
    assert checked > 30
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
        assert reports[p] == want, f"request {p}"
        o = ref.outcome
        assert outcomes[p]["final"] == o.final and outcomes[p]["reason"] == o.termination_reason
        assert outcomes[p]["tally"] == o.tally
        assert outcomes[p]["tokens_decode"] == o.tokens_decode


def test_fused_step_steady_state_matches_split_kernels():
    """Cycling pool (the bench workload shape): per-round totals of the fused
    step equal those of the split launches (advance / K1 / round), since the
    same requests are admitted each round and each evolves independently."""
    from paper_2509_24957_b200 import _lib
    from paper_2509_24957_b200.engine import BatchedDuchess
    from paper_2509_24957_b200.probe import ProbeBank, Scorer, fill_windows
    knobs, traces, seeds = _setup(96, 16, 0.8)
    R, C, L, T, H = 32, 16, 1, 4, 512
    w, g, beta = _probe(H, L)
    bank = ProbeBank.from_linear(w, np.zeros(L), g, beta)

    def make():
        return BatchedDuchess(traces, knobs, seeds, n_slots=R, pred_source=_lib.PRED_DEVICE,
                              queue=list(range(len(traces))), cycle=True)
    a, b = make(), make()
    acts = torch.zeros((R * C, L, T, H), dtype=torch.bfloat16, device="cuda")
    logit = torch.zeros(R * C * L, device="cuda")
    scorer = Scorer(bank, R * C * L)
    a.advance()
    b.begin_fused()
    for step in range(60):
        fill_windows(acts, 9, a.t["row_req"], a.t["row_tmpl"], a.t["row_pos"], a.t["row_mask"])
        scorer.score_active(acts, logit.view(R * C, L), a.probs.view(R * C, L), a)
        a.round()
        fill_windows(acts, 9, b.t["row_req"], b.t["row_tmpl"], b.t["row_pos"], b.t["row_mask"])
        b.step_fused(acts, bank, logit)
        ra = sorted((p, rep) for p, rep in a.round_reports())
        rb = sorted((p, rep) for p, rep in b.round_reports())
        assert ra == rb, f"step {step}"
    assert (a.counters()[:5] == b.counters()[:5]).all()


def test_upload_survivors_copies_only_listed_rows():
    """duchess_gather_active: exactly the rows of the round in flight's active
    list (either parity) arrive from pinned host memory; others untouched."""
    from paper_2509_24957_b200 import _lib
    from paper_2509_24957_b200.engine import BatchedDuchess
    knobs, traces, seeds = _setup(40, 8, 1.0)
    R, C = 6, 8
    eng = BatchedDuchess(traces, knobs, seeds, n_slots=R, pred_source=_lib.PRED_DEVICE,
                         queue=list(range(len(traces))), cycle=True)
    host = torch.randint(-1000, 1000, (R * C, 1, 3, 64), dtype=torch.int16).view(
        torch.bfloat16).pin_memory()
    eng.advance()
    for step in range(6):
        dev = torch.zeros_like(host, device="cuda")
        eng.upload_survivors(host, dev)
        torch.cuda.synchronize()
        mask = eng.t["row_mask"].cpu().numpy().astype(bool)
        d = dev.cpu().view(torch.int16)
        h = host.view(torch.int16)
        assert mask.any()
        assert torch.equal(d[torch.from_numpy(mask)], h[torch.from_numpy(mask)])
        assert not d[torch.from_numpy(~mask)].any()
        eng.probs.fill_(0.5)
        eng.round()
