"""K2 parity on the GPU: the batched decision engine must reproduce the
reference's DuchessRun round by round, bit-exact, for every golden case
(decisions.json, made by running the reference), with fewer device slots than
requests so finished slots are refilled on device from the service queue."""

import random

import numpy as np
import pytest
import torch

from oracle import activations as oact
from oracle import port
from tests.golden_util import (STATUS, case_knobs, case_traces, load, port_report_tuple,
                               report_tuple)

pytestmark = pytest.mark.gpu


def run_engine(engine, max_steps=100000, on_step=None):
    from paper_2509_24957_b200 import _lib
    reports: dict[int, list] = {}
    branches: dict[int, list] = {}
    for _ in range(max_steps):
        engine.step()
        for p, rep in engine.round_reports():
            reports.setdefault(p, []).append(rep)
            if rep[6]:
                slot = int(np.nonzero(engine.t["slot_req"].cpu().numpy() == p)[0][0])
                snap = engine.branch_snapshot(slot)
                ans = engine.wl.answers[p]
                branches[p] = [[STATUS[int(s)], None if f < 0 else ans[int(f)], int(ob), int(td),
                                int(st), int(n), float(lp).hex()]
                               for s, f, ob, td, st, n, lp in zip(
                                   snap["br_status"], snap["br_final"], snap["br_offset"],
                                   snap["br_decoded"], snap["br_streak"], snap["br_npred"],
                                   snap["br_last_pred"])]
        if on_step:
            on_step(engine)
        if engine.all_done():
            break
    assert int(engine.counters()[_lib.CNT_AMBIGUOUS]) == 0
    return reports, branches


@pytest.mark.parametrize("case", load("decisions.json"), ids=lambda c: c["name"])
@pytest.mark.parametrize("slots,reverse", [(5, False), (64, True)])
def test_engine_matches_reference_golden(case, slots, reverse):
    from paper_2509_24957_b200 import _lib
    from paper_2509_24957_b200.engine import BatchedDuchess
    traces = case_traces(case)
    knobs = case_knobs(case)
    seeds = [int(r["seed"]) for r in case["requests"]]
    n = len(traces)
    queue = list(range(n))[::-1] if reverse else list(range(n))
    eng = BatchedDuchess(traces, knobs, seeds, n_slots=min(slots, n),
                         pred_source=_lib.PRED_TRACE, rho=case["rho"], queue=queue)
    reports, branches = run_engine(eng)
    outcomes = eng.outcomes()
    for p, ref in enumerate(case["requests"]):
        assert reports[p] == [report_tuple(r) for r in ref["reports"]], f"request {p}"
        o = outcomes[p]
        assert (o["tally"], o["final"], o["reason"], o["tokens_decode"], o["tokens_probe"],
                o["rounds"]) == (ref["outcome"]["tally"], ref["outcome"]["final"],
                                 ref["outcome"]["reason"], ref["outcome"]["tokens_decode"],
                                 ref["outcome"]["tokens_probe"], ref["outcome"]["rounds"])
        want = [[STATUS[s], fa, ob, td, st, npred, lp]
                for s, fa, ob, td, st, npred, lp in ref["branches"]]
        assert branches[p] == want, f"request {p} branch states"


@pytest.mark.parametrize("case", load("decisions.json"), ids=lambda c: c["name"])
@pytest.mark.parametrize("exact_cdf", [False, True])
def test_fused_round_kernel_matches_reference_golden(case, exact_cdf):
    """duchess_round (decide k + advance k+1 in one cooperative launch) must
    give the same RoundReports and outcomes as the split kernels."""
    from paper_2509_24957_b200 import _lib
    from paper_2509_24957_b200.engine import BatchedDuchess
    traces = case_traces(case)
    seeds = [int(r["seed"]) for r in case["requests"]]
    eng = BatchedDuchess(traces, case_knobs(case), seeds, n_slots=min(7, len(traces)),
                         pred_source=_lib.PRED_TRACE, rho=case["rho"])
    if exact_cdf:
        eng.policy.flags |= _lib.FLAG_EXACT_CDF
    eng.advance()
    reports = {}
    for _ in range(100000):
        eng.round()
        for p, rep in eng.round_reports():
            reports.setdefault(p, []).append(rep)
        if eng.all_done():
            break
    outcomes = eng.outcomes()
    for p, ref in enumerate(case["requests"]):
        assert reports[p] == [report_tuple(r) for r in ref["reports"]], f"request {p}"
        assert outcomes[p]["final"] == ref["outcome"]["final"]
        assert outcomes[p]["tally"] == ref["outcome"]["tally"]
        assert outcomes[p]["tokens_decode"] == ref["outcome"]["tokens_decode"]


def _c1_setup(n_req=24, templates=64, c=8, temperature=1.0):
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


@pytest.mark.parametrize("dtype,T,temperature", [(torch.float32, 1, 1.0),
                                                 (torch.bfloat16, 32, 0.8)])
def test_scores_to_decisions_composition(dtype, T, temperature):
    """K1 probabilities -> K2 decisions == oracle DuchessRun fed the same
    probabilities through predictor= (the reference seam,
    orchestrator.py:319-327, :358-363); logits within 1e-4*max(|ref|,1) of the
    fp64 oracle on the regenerated windows."""
    from paper_2509_24957_b200 import _lib
    from paper_2509_24957_b200.engine import BatchedDuchess
    from paper_2509_24957_b200.probe import ProbeBank, Scorer, fill_windows
    H, L, seed = 4096, 1, 1
    knobs, traces, seeds = _c1_setup(temperature=temperature)
    rng = np.random.default_rng(0)
    w = rng.normal(0.0, 1.5 / np.sqrt(H), size=(1, H))
    g = rng.uniform(0.5, 1.5, size=(1, H))
    beta = rng.uniform(-0.1, 0.1, size=(1, H))
    bank = ProbeBank.from_linear(w, [0.0], g, beta)
    R = 8
    eng = BatchedDuchess(traces, knobs, seeds, n_slots=R, pred_source=_lib.PRED_DEVICE)
    C = knobs.max_branches
    acts = torch.zeros((R * C, L, T, H), dtype=dtype, device="cuda")
    scorer = Scorer(bank, R * C * L)
    logit = torch.zeros((R * C, L), device="cuda")
    seen = {}
    checked = [0]

    def score(e):
        t = e.t
        fill_windows(acts, seed, t["row_req"], t["row_tmpl"], t["row_pos"], t["row_mask"])
        scorer(acts, logit, e.probs.view(R * C, L), row_mask=t["row_mask"])

    def record(e):
        t = e.t
        mask = t["row_mask"].cpu().numpy().astype(bool)
        req = t["row_req"].cpu().numpy()
        tm = t["row_tmpl"].cpu().numpy()
        pos = t["row_pos"].cpu().numpy()
        pr = e.probs.cpu().numpy()
        lg = logit.cpu().numpy()[:, 0]
        for row in np.nonzero(mask)[0]:
            key = (int(req[row]), int(tm[row]), int(pos[row]))
            seen[key] = float(pr[row])
            if checked[0] < 200 and row % 3 == 0:
                win = oact.synth_window(seed, *key, 0, T, H, dtype == torch.bfloat16)
                ref, _ = port.pooled_linear_probe(win, w[0], 0.0, g[0], beta[0])
                assert abs(float(lg[row]) - ref) <= 1e-4 * max(abs(ref), 1.0)
                checked[0] += 1

    reports = {}
    for _ in range(10000):
        eng.step(score_fn=score)
        record(eng)
        for p, rep in eng.round_reports():
            reports.setdefault(p, []).append(rep)
        if eng.all_done():
            break
    assert checked[0] > 50
    assert int(eng.counters()[_lib.CNT_AMBIGUOUS]) == 0
    outcomes = eng.outcomes()
    for p, trace in enumerate(traces):
        index = {id(t): j for j, t in enumerate(trace.templates)}

        def predictor(tmpl, position, _rng, p=p, index=index):
            return seen[(p, index[id(tmpl)], position)]

        req = port.DuchessRequest(trace, knobs, random.Random(seeds[p]), predictor=predictor)
        want = []
        while not req.done:
            want.append(port_report_tuple(req.step()))
        assert reports[p] == want, f"request {p}"
        o = req.outcome
        assert outcomes[p]["final"] == o.final and outcomes[p]["reason"] == o.termination_reason
        assert outcomes[p]["tally"] == o.tally


def test_probe_lookup_long_probe_lists():
    """8-ary probe_answer search vs the oracle's bisect on templates with up to
    600 probes, convergence points, and positions on/around every boundary."""
    from paper_2509_24957_b200 import _lib
    from paper_2509_24957_b200.engine import pack_workload
    rng = random.Random(12)
    traces, queries = [], []
    for i in range(40):
        n_probes = rng.choice([0, 1, 2, 7, 8, 9, 17, 64, 65, 200, 600])
        ats = sorted(rng.sample(range(1, 5000), n_probes))
        length = (ats[-1] if ats else 10) + rng.randint(0, 50)
        conv = rng.choice([None, rng.randint(0, length)])
        probes = [(a, str(rng.randint(0, 30))) for a in ats]
        if conv is not None:
            probes = [(a, "f" if a >= conv else x) for a, x in probes]
        t = port.Tmpl(length, "f", probes, conv)
        traces.append(port.Trace(f"q{i}", "f", 0, [t]))
        pts = {0, length, length + 3}
        for a in ats[:50] + ats[-50:]:
            pts.update({a - 1, a, a + 1})
        queries.append(sorted(p for p in pts if p >= 0))
    wl = pack_workload(traces, [[0] * _lib.MT_WORDS] * len(traces), list(range(len(traces))),
                       False, torch.device("cuda"))
    tm, ps, want = [], [], []
    for i, (tr, qs) in enumerate(zip(traces, queries)):
        for q in qs:
            tm.append(i)
            ps.append(q)
            want.append(wl.answers[i].index(port.probe_answer(tr.templates[0], q)))
    lib = _lib.load()
    t_ = torch.tensor(tm, dtype=torch.int32, device="cuda")
    p_ = torch.tensor(ps, dtype=torch.int32, device="cuda")
    out = torch.empty(len(tm), dtype=torch.int32, device="cuda")
    _lib.check(lib.duchess_template_lookup(wl.struct, t_.data_ptr(), p_.data_ptr(), len(tm),
                                           out.data_ptr(), None, _lib.stream_handle()), "lookup")
    assert out.cpu().tolist() == want


@pytest.mark.parametrize("case", load("baselines.json"), ids=lambda c: c["name"])
def test_baseline_policies_match_reference_golden(case):
    """Default SC / Short-m@k / Dynasor on the device engine (slot refill on)
    vs the reference's own runs (tests/golden/baselines.json)."""
    from paper_2509_24957_b200.engine import BatchedDuchess
    from tests.golden_util import gen_params
    traces = port.generate(gen_params(case["params"]), case["n"], case["workload_seed"])
    eng = BatchedDuchess(traces, case_knobs(case), [0] * len(traces), n_slots=6,
                         policy=case["policy"])
    reports = {}
    for _ in range(100000):
        eng.step()
        for p, rep in eng.round_reports():
            reports.setdefault(p, []).append(rep)
        if eng.all_done():
            break
    outcomes = eng.outcomes()
    for p, ref in enumerate(case["requests"]):
        assert reports[p] == [report_tuple(r) for r in ref["reports"]], f"request {p}"
        o = outcomes[p]
        assert (o["tally"], o["final"], o["reason"], o["tokens_decode"], o["tokens_probe"],
                o["rounds"]) == tuple(ref["outcome"][k] for k in (
                    "tally", "final", "reason", "tokens_decode", "tokens_probe", "rounds"))
