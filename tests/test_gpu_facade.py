"""The reference-facing API (paper_2509_24957_b200.*) on the GPU: the
reference's own round-level and rule tests (pkg/tests/test_orchestrator.py,
test_core.py, test_predictor.py, test_scheduler.py, test_workload.py) restated
against the device-backed facade, plus the golden primitive fixtures made by
running the reference (tests/golden/primitives.json)."""

import random

import numpy as np
import pytest

from oracle import port
from tests.golden_util import fx, load

pytestmark = pytest.mark.gpu


def small_config(**kw):
    from paper_2509_24957_b200.orchestrator import OrchestratorConfig
    d = dict(max_branches=2, interval_tokens=16, early_term_threshold=0.5, early_term_rounds=1,
             branch_out_temperature=1.0, consensus_frac=0.6, coverage_frac=0.8, token_cap=4096,
             probe_cost_tokens=10)
    d.update(kw)
    return OrchestratorConfig(**d)


def tmpl(length, final, probes=(), conv=None, pred=None):
    from paper_2509_24957_b200.workload import BranchTemplate
    return BranchTemplate(length, final, [tuple(p) for p in probes], conv,
                          [tuple(p) for p in pred] if pred is not None else None)


def trace(gt, templates):
    from paper_2509_24957_b200.workload import RequestTrace
    return RequestTrace("t", gt, 0, list(templates))


# ---- rule primitives (test_orchestrator.py:41-138) -------------------------

def test_early_termination_rule():
    from paper_2509_24957_b200.orchestrator import BranchState, check_early_termination

    def br(h):
        b = BranchState(0, 0, tmpl(100, "x"))
        b.prediction_history = list(h)
        return b
    assert check_early_termination(br([0.9, 0.92]), 0.85, 2)
    assert not check_early_termination(br([0.9, 0.7, 0.9]), 0.85, 2)
    assert not check_early_termination(br([0.9]), 0.85, 2)
    assert not check_early_termination(br([0.85, 0.85]), 0.85, 2)


def test_branch_out_known_answers():
    from paper_2509_24957_b200.orchestrator import branch_out_sample, branch_out_weights
    assert branch_out_weights([0.8, 0.2], 1.0) == pytest.approx([0.8, 0.2])
    assert branch_out_weights([0.8, 0.2], 0.5) == pytest.approx([0.9412, 0.0588], abs=1e-4)
    for t in (0.3, 0.8, 1.0, 2.5):
        assert branch_out_weights([0.5, 0.5], t) == pytest.approx([0.5, 0.5])
    w = branch_out_weights([0.0, 1.0], 0.5)
    assert w[0] > 0 and w[1] == pytest.approx(1.0, abs=1e-9)
    with pytest.raises(ValueError, match="no branch to duplicate"):
        branch_out_weights([], 1.0)
    with pytest.raises(ValueError, match="no branch to duplicate"):
        branch_out_sample([], 1.0, random.Random(0))


def test_branch_out_golden_fixture():
    from paper_2509_24957_b200.orchestrator import (branch_out_sample, branch_out_sample_many,
                                                    branch_out_weights)
    for i, case in enumerate(load("primitives.json")["branch_out"]):
        probs = [fx(p) for p in case["probs"]]
        temp = fx(case["temperature"])
        w = branch_out_weights(probs, temp)
        np.testing.assert_allclose(w, [fx(x) for x in case["weights"]], rtol=1e-14, atol=0)
        if temp == 1.0:
            assert [x.hex() for x in w] == case["weights"]
        if i % 10 == 0:
            assert [branch_out_sample(probs, temp, random.Random(s)) for s in range(8)] == \
                case["draws"]
        rng = random.Random(case["seq_seed"])
        assert branch_out_sample_many(probs, temp, rng, 20) == case["seq"]
        # the caller's rng advanced exactly like the reference's
        ref = random.Random(case["seq_seed"])
        for _ in range(20):
            ref.random()
        assert rng.random() == ref.random()


def test_request_termination_rules():
    from paper_2509_24957_b200.core import VoteTally
    from paper_2509_24957_b200.orchestrator import check_request_termination as crt
    assert crt(VoteTally(["a"] * 6), 0.6, 0.8, 10) == "consensus"
    assert crt(VoteTally(["a"] * 4 + ["b"] * 4), 0.6, 0.8, 10) == "coverage"
    assert crt(VoteTally(["a"] * 5 + ["b"] * 2), 0.6, 0.8, 10) is None
    assert crt(VoteTally(["a"] * 8), 0.6, 0.8, 10) == "consensus"
    rng = random.Random(4)
    for _ in range(50):
        t = VoteTally([str(rng.randrange(4)) for _ in range(rng.randrange(12))])
        assert crt(t, 0.6, 0.8, 10) == port.request_termination(dict(t.counts), 0.6, 0.8, 10)


def test_majority_vote():
    from paper_2509_24957_b200.core import VoteTally, majority_vote
    assert majority_vote(VoteTally(["a", "a", "b"])) == "a"
    assert majority_vote(VoteTally(["a", "b"])) == "a"
    assert majority_vote(VoteTally(["b", "a"])) == "a"
    assert majority_vote(VoteTally(["", "x"])) == ""
    with pytest.raises(ValueError, match="no answers collected"):
        majority_vote(VoteTally())
    rng = random.Random(9)
    for _ in range(30):
        ans = [rng.choice(["3", "12", "7", "", "b"]) for _ in range(rng.randint(1, 9))]
        assert majority_vote(VoteTally(ans)) == port.majority_vote(dict(VoteTally(ans).counts))


# ---- round-level hand traces (test_orchestrator.py:145-248) ----------------

def test_round_continues_below_threshold():
    from paper_2509_24957_b200.orchestrator import DuchessRun
    from paper_2509_24957_b200.predictor import SyntheticPredictorConfig
    run = DuchessRun(trace("9", [tmpl(400, "9", conv=300) for _ in range(2)]), small_config(),
                     random.Random(0), synthetic=SyntheticPredictorConfig(rho=1.0))
    rep = run.step()
    assert [a.kind for a in rep.actions] == ["continue", "continue"]
    assert run.tokens_decode == 32
    assert all(b.tokens_decoded == 16 for b in run.branches)
    assert not run.done


def test_single_branch_consensus_hand_trace():
    from paper_2509_24957_b200.orchestrator import CONSENSUS, DuchessRun
    from paper_2509_24957_b200.predictor import SyntheticPredictorConfig
    run = DuchessRun(trace("9", [tmpl(64, "9", conv=10)]),
                     small_config(max_branches=1, early_term_threshold=0.9), random.Random(0),
                     synthetic=SyntheticPredictorConfig(rho=1.0))
    rep = run.step()
    assert rep.done
    o = run.outcome
    assert (o.termination_reason, o.tokens_decode, o.tokens_probe, o.tokens_total, o.rounds,
            o.final) == (CONSENSUS, 16, 10, 26, 1, "9")
    with pytest.raises(RuntimeError, match="request already terminated"):
        run.step()


def test_natural_end_and_capped():
    from paper_2509_24957_b200.orchestrator import (CAPPED, NATURAL_END, TERMINATION_DISABLED,
                                                    DuchessRun)
    run = DuchessRun(trace("9", [tmpl(40, "9")]),
                     small_config(max_branches=1, early_term_threshold=TERMINATION_DISABLED,
                                  consensus_frac=1.0, coverage_frac=1.0), random.Random(0))
    o = run.run()
    assert (o.tokens_probe, o.tokens_decode, run.branches[0].status, o.rounds) == \
        (0, 40, NATURAL_END, 3)
    run = DuchessRun(trace("9", [tmpl(100, "9", conv=50)]),
                     small_config(max_branches=1, token_cap=64,
                                  early_term_threshold=TERMINATION_DISABLED,
                                  consensus_frac=1.0, coverage_frac=1.0), random.Random(0))
    o = run.run()
    b = run.branches[0]
    assert (b.status, b.tokens_decoded, o.tokens_probe, o.final) == (CAPPED, 64, 10, "9")
    assert b.probe_history == [(64, "9")]


def test_fork_inherits_position_and_resets_history():
    from paper_2509_24957_b200.orchestrator import EARLY_TERMINATED, DuchessRun
    from paper_2509_24957_b200.predictor import SyntheticPredictorConfig
    run = DuchessRun(trace("9", [tmpl(600, "9", conv=40), tmpl(600, "5", conv=300),
                                 tmpl(600, "9", conv=100)]),
                     small_config(consensus_frac=1.0, coverage_frac=1.0), random.Random(0),
                     synthetic=SyntheticPredictorConfig(rho=1.0))
    reports = []
    while not run.done:
        reports.append(run.step())
    forks = [a for r in reports for a in r.actions if a.kind == "branch_out"]
    assert len(forks) == 1
    child = run.branches[forks[0].branch_id]
    assert child.offset_base == 48 and child.template_index == 2
    assert child.prediction_history == [0.0, 0.0, 0.0, 1.0]
    assert child.status == EARLY_TERMINATED and child.final_answer == "9"
    assert run.tokens_decode == sum(b.tokens_decoded for b in run.branches)


def test_fork_clamped_to_template_end():
    from paper_2509_24957_b200.orchestrator import NATURAL_END, DuchessRun
    from paper_2509_24957_b200.predictor import SyntheticPredictorConfig
    run = DuchessRun(trace("9", [tmpl(64, "9"), tmpl(400, "5", conv=399), tmpl(30, "7")]),
                     small_config(consensus_frac=1.0, coverage_frac=1.0,
                                  early_term_threshold=0.9), random.Random(0),
                     synthetic=SyntheticPredictorConfig(rho=1.0))
    run.run()
    child = next(b for b in run.branches if b.template_index == 2)
    assert (child.offset_base, child.tokens_decoded, child.status, child.final_answer) == \
        (30, 0, NATURAL_END, "7")


def test_facade_replays_oracle_and_advances_rng():
    """Random synthetic workloads: facade == oracle port, including the rng
    stream left behind (shared rng across consecutive runs)."""
    from paper_2509_24957_b200.orchestrator import DuchessRun, OrchestratorConfig
    from paper_2509_24957_b200.predictor import SyntheticPredictorConfig
    from paper_2509_24957_b200.workload import SyntheticParams, generate_synthetic
    wl = generate_synthetic(SyntheticParams(templates_per_request=15), 6, seed=3)
    cfg = OrchestratorConfig(max_branches=6, interval_tokens=80, early_term_threshold=0.6,
                             early_term_rounds=1, branch_out_temperature=0.7)
    knobs = port.Knobs(max_branches=6, interval_tokens=80, early_term_threshold=0.6,
                       early_term_rounds=1, branch_out_temperature=0.7)
    rng_a, rng_b = random.Random(5), random.Random(5)
    for tr in wl.requests:
        a = DuchessRun(tr, cfg, rng_a, synthetic=SyntheticPredictorConfig(rho=0.7))
        b = port.DuchessRequest(tr, knobs, rng_b, rho=0.7)
        while not a.done:
            ra, rb = a.step(), b.step()
            assert (ra.round_index, ra.decoding_branches, ra.max_chunk, ra.decode_tokens,
                    ra.probes, [(x.kind, x.branch_id, x.source_branch_id) for x in ra.actions],
                    ra.done) == (rb.round_index, rb.decoding_branches, rb.max_chunk,
                                 rb.decode_tokens, rb.probes, rb.actions, rb.done)
        assert b.done
        assert a.outcome.final == b.outcome.final
        assert dict(a.outcome.tally.counts) == b.outcome.tally
        for x, y in zip(a.branches, b.branches):
            assert (x.status, x.final_answer, x.offset_base, x.tokens_decoded, x.streak,
                    x.prediction_history, x.last_prediction) == \
                (y.status, y.final_answer, y.offset_base, y.tokens_decoded, y.streak,
                 y.prediction_history, y.last_prediction)
    assert rng_a.getstate() == rng_b.getstate()


def test_host_predictor_seam():
    """A user predictor= callable is honoured (called per survivor in creation
    order, may draw from the rng) exactly like the reference seam."""
    from paper_2509_24957_b200.orchestrator import DuchessRun, OrchestratorConfig
    from paper_2509_24957_b200.workload import SyntheticParams, generate_synthetic
    wl = generate_synthetic(SyntheticParams(templates_per_request=12), 4, seed=8)
    cfg = OrchestratorConfig(max_branches=5, interval_tokens=40, early_term_threshold=0.55)
    knobs = port.Knobs(max_branches=5, interval_tokens=40, early_term_threshold=0.55)
    for tr in wl.requests:
        calls_a, calls_b = [], []

        def mk(calls):
            def pred(template, position, rng):
                calls.append((template.natural_length, position))
                return (rng.random() + (position % 7) / 7.0) / 2.0
            return pred
        a = DuchessRun(tr, cfg, random.Random(1), predictor=mk(calls_a))
        b = port.DuchessRequest(tr, knobs, random.Random(1), predictor=mk(calls_b))
        while not a.done:
            ra, rb = a.step(), b.step()
            assert [(x.kind, x.branch_id, x.source_branch_id) for x in ra.actions] == rb.actions
        assert calls_a == calls_b
        assert a.outcome.final == b.outcome.final


def test_active_branch_count_never_exceeds_limit():
    from paper_2509_24957_b200.orchestrator import ACTIVE, DuchessRun, OrchestratorConfig
    from paper_2509_24957_b200.predictor import SyntheticPredictorConfig
    from paper_2509_24957_b200.workload import SyntheticParams, generate_synthetic
    wl = generate_synthetic(SyntheticParams(templates_per_request=15), 4, seed=3)
    cfg = OrchestratorConfig(max_branches=6, interval_tokens=80, early_term_threshold=0.5,
                             early_term_rounds=1)
    for i, tr in enumerate(wl.requests):
        run = DuchessRun(tr, cfg, random.Random(i), synthetic=SyntheticPredictorConfig(rho=1.0))
        while not run.done:
            run.step()
            active = [b for b in run.branches if b.status == ACTIVE]
            assert len(active) <= cfg.max_branches
            if not run.done and run._next_template < len(tr.templates):
                assert len(active) == cfg.max_branches



def test_early_terminated_branches_satisfy_rule_and_replay_is_deterministic():
    """test_orchestrator.py:267-296: every early-terminated branch held the
    threshold for the last early_term_rounds predictions, streak <= history;
    two runs with equal seeds give equal RoundReports and outcomes."""
    from paper_2509_24957_b200.orchestrator import EARLY_TERMINATED, DuchessRun, OrchestratorConfig
    from paper_2509_24957_b200.predictor import SyntheticPredictorConfig
    from paper_2509_24957_b200.workload import SyntheticParams, generate_synthetic
    wl = generate_synthetic(SyntheticParams(), 10, seed=5)
    cfg = OrchestratorConfig(max_branches=10, interval_tokens=80, early_term_threshold=0.5,
                             early_term_rounds=2)
    for i, tr in enumerate(wl.requests):
        run = DuchessRun(tr, cfg, random.Random(i), synthetic=SyntheticPredictorConfig(rho=1.0))
        run.run()
        for b in run.branches:
            if b.status == EARLY_TERMINATED:
                assert len(b.prediction_history) >= 2
                assert all(p > 0.5 for p in b.prediction_history[-2:])
            assert b.streak <= len(b.prediction_history)
    wl = generate_synthetic(SyntheticParams(), 5, seed=6)
    cfg = OrchestratorConfig(early_term_threshold=0.6, early_term_rounds=1)
    synth = SyntheticPredictorConfig(rho=0.7)
    for i, tr in enumerate(wl.requests):
        a = DuchessRun(tr, cfg, random.Random(i), synthetic=synth)
        b = DuchessRun(tr, cfg, random.Random(i), synthetic=synth)
        ra, rb = [], []
        while not a.done:
            ra.append(a.step())
        while not b.done:
            rb.append(b.step())
        assert ra == rb and a.outcome == b.outcome


def test_policy_reduction_matches_default_sc():
    """test_orchestrator.py:299-313: with termination disabled and full
    consensus / coverage bounds the policy is plain self-consistency."""
    from paper_2509_24957_b200.orchestrator import (TERMINATION_DISABLED, OrchestratorConfig,
                                                    run_default_sc, run_duchess)
    from paper_2509_24957_b200.workload import SyntheticParams, generate_synthetic
    wl = generate_synthetic(SyntheticParams(templates_per_request=8), 30, seed=7)
    cfg = OrchestratorConfig(max_branches=8, interval_tokens=80,
                             early_term_threshold=TERMINATION_DISABLED, consensus_frac=1.0,
                             coverage_frac=1.0)
    for i, tr in enumerate(wl.requests):
        sc, du = run_default_sc(tr, cfg), run_duchess(tr, cfg, random.Random(i))
        assert (du.tokens_decode, du.tokens_probe, du.tally, du.final) == \
            (sc.tokens_decode, sc.tokens_probe, sc.tally, sc.final)

# ---- predictor (test_predictor.py) + golden fixture -------------------------

def _mlp(case):
    from paper_2509_24957_b200.predictor import MlpWeights
    dims = [case["input_dim"], *case["layer_dims"], case["head_dim"]]
    bn = case["bn"]
    return MlpWeights(
        case["input_dim"], case["layer_dims"], case["head_dim"], case["activations"],
        [np.array([fx(v) for v in m]).reshape(dims[k + 1], dims[k])
         for k, m in enumerate(case["weights"])],
        [np.array([fx(v) for v in b]) for b in case["biases"]],
        None if case["ln_gain"] is None else np.array([fx(v) for v in case["ln_gain"]]),
        None if case["ln_bias"] is None else np.array([fx(v) for v in case["ln_bias"]]),
        *([None] * 4 if bn is None else
          [[np.array([fx(v) for v in vec]) for vec in part] for part in bn]))


def test_mlp_forward_golden():
    from paper_2509_24957_b200.predictor import mlp_forward
    for case in load("primitives.json")["mlp"]:
        logits, probs = mlp_forward(_mlp(case), [fx(v) for v in case["x"]])
        np.testing.assert_allclose(logits, [fx(v) for v in case["logits"]], atol=1e-10)
        np.testing.assert_allclose(probs, [fx(v) for v in case["probs"]], atol=1e-10)


def test_mlp_forward_errors_and_zero_net():
    from paper_2509_24957_b200.predictor import MlpWeights, WeightFormatError, mlp_forward
    z = MlpWeights(8, [4, 3], 1, ["relu", "relu"],
                   [np.zeros((4, 8)), np.zeros((3, 4)), np.zeros((1, 3))],
                   [np.zeros(4), np.zeros(3), np.zeros(1)], np.ones(8), np.zeros(8))
    assert mlp_forward(z, np.arange(8.0))[1][0] == pytest.approx(0.5)
    with pytest.raises(WeightFormatError, match=r"\(7,\).*\(8,\)"):
        mlp_forward(z, np.zeros(7))


def test_weight_round_trip_including_linear_probe(tmp_path):
    from paper_2509_24957_b200.predictor import load_weights, mlp_forward, save_weights
    case = load("primitives.json")["mlp"][0]
    rng = np.random.default_rng(0)
    for w in (_mlp(case), _linear(rng)):
        save_weights(w, tmp_path / "p.mlp")
        back = load_weights(tmp_path / "p.mlp")
        x = rng.uniform(-1, 1, w.input_dim)
        assert mlp_forward(back, x)[1] == pytest.approx(mlp_forward(w, x)[1], abs=1e-5)


def _linear(rng):
    from paper_2509_24957_b200.predictor import MlpWeights
    return MlpWeights(16, [], 1, [], [rng.normal(size=(1, 16))], [np.array([0.1])],
                      rng.uniform(0.5, 1.5, 16), rng.uniform(-0.1, 0.1, 16))


def test_synthetic_predict_and_confusion_match_reference_streams():
    from paper_2509_24957_b200.predictor import (DEFAULT_CONFUSION, SyntheticPredictorConfig,
                                                 predict_difficulty, sample_confused_level,
                                                 synthetic_predict)
    for case in load("primitives.json")["confusion"]:
        rng = random.Random(case["seed"])
        assert [sample_confused_level(case["level"], DEFAULT_CONFUSION, rng)
                for _ in range(10)] == case["seq"][:10]
    r1, r2 = random.Random(3), random.Random(3)
    for k in range(20):
        cfg = SyntheticPredictorConfig(rho=k / 19)
        assert synthetic_predict(k % 2 == 0, cfg, r1) == port.synthetic_predict(k % 2 == 0,
                                                                                cfg.rho, r2)
    assert r1.getstate() == r2.getstate()
    assert predict_difficulty("actual", actual_label=3) == 3
    with pytest.raises(ValueError, match="unknown difficulty mode"):
        predict_difficulty("nope")


# ---- scheduler / workload ----------------------------------------------------

def test_next_request_golden_orders():
    from paper_2509_24957_b200.scheduler import EASIEST_ACTUAL, FCFS, QueueEntry, next_request
    from paper_2509_24957_b200.workload import BranchTemplate, RequestTrace
    for case in load("primitives.json")["orders"][:30]:
        n = len(case["levels"])
        traces = [RequestTrace(f"q{j}", "1", 0, [BranchTemplate(10, "1")], case["levels"][j])
                  for j in range(n)]
        q = [QueueEntry(traces[j], case["arrivals"][j], j) for j in case["insert"]]
        got = []
        while q:
            got.append(next_request(q, case["policy"], 10 ** 9).order)
        assert got == case["order"]
    with pytest.raises(ValueError, match="no eligible request"):
        next_request([], FCFS, 0)
    del EASIEST_ACTUAL


def test_next_request_ties_and_wide_fields_match_reference_scan():
    """Duplicate (level, arrival, order) tuples keep the first queue entry
    (the reference's strict `<` scan, scheduler.py:91-93); negative, large
    and > 7 levels go through the rank-packed keys."""
    from paper_2509_24957_b200.scheduler import EASIEST_ACTUAL, FCFS, QueueEntry, next_request
    from paper_2509_24957_b200.workload import BranchTemplate, RequestTrace

    def ref_pick(q, policy):
        best, bk = -1, None
        for i, e in enumerate(q):
            k = ((e.arrival, e.order) if policy == FCFS
                 else (e.trace.difficulty, e.arrival, e.order))
            if bk is None or k < bk:
                best, bk = i, k
        return best

    rng = random.Random(9)
    for case in range(40):
        n = rng.randint(1, 24)
        wide = case % 2 == 1
        q = []
        for j in range(n):
            lv = rng.choice([-3, 0, 9, 2 ** 40]) if wide else rng.randint(1, 3)
            ar = rng.choice([0, 5, 2 ** 45]) if wide else rng.randint(0, 3)
            od = rng.choice([0, 1, 2 ** 30]) if wide else rng.randint(0, 2)
            q.append(QueueEntry(RequestTrace(f"q{j}", "1", 0, [BranchTemplate(10, "1")], lv),
                                ar, od))
        policy = FCFS if case % 3 == 0 else EASIEST_ACTUAL
        qr = list(q)
        while q:
            want = qr.pop(ref_pick(qr, policy))
            assert next_request(q, policy, 2 ** 50) is want


def test_difficulty_queue_large_pool_matches_sorted():
    from paper_2509_24957_b200.scheduler import difficulty_queue
    rng = random.Random(2)
    for n in (1, 17, 4096, 10000):
        levels = [rng.randint(1, 5) for _ in range(n)]
        arrivals = sorted(rng.randrange(10 ** 9) for _ in range(n))
        want = sorted(range(n), key=lambda j: (levels[j], arrivals[j], j))
        assert difficulty_queue(levels, arrivals) == want


def test_device_sort_merge_passes_any_size_stable():
    """duchess_sort_keys (4096-key tiles + merge-path passes) equals a stable
    host sort for sizes around the tile / pass boundaries, with many equal keys
    (ties keep input order, like the reference's first-in-queue pick)."""
    from paper_2509_24957_b200.scheduler import device_sort
    rng = np.random.default_rng(5)
    for n in (4097, 8191, 8192, 12289, 65536 + 3, 300001):
        keys = rng.integers(0, max(2, n // 7), size=n, dtype=np.uint64) << np.uint64(20)
        got = device_sort(keys)
        want = np.argsort(keys, kind="stable").tolist()
        assert got == want, n


def test_probe_answer_and_trace_prediction():
    from paper_2509_24957_b200.workload import probe_answer, trace_prediction
    t = tmpl(100, "42", probes=[(16, "7"), (32, "13")], conv=64)
    assert [probe_answer(t, p) for p in (8, 16, 40, 90, 200)] == ["", "7", "13", "42", "42"]
    t = tmpl(100, "1", pred=[(16, 0.25), (32, 0.75)])
    assert [trace_prediction(t, p) for p in (10, 20, 32)] == [0.0, 0.25, 0.75]


def test_baseline_facades_match_reference_behaviour():
    """The reference's baseline tests (test_orchestrator.py:337-460,
    test_acceptance.py crit 1 and 10) against the device-backed facades."""
    from paper_2509_24957_b200.orchestrator import (CANCELLED, DefaultScRun, DynasorRun,
                                                    OrchestratorConfig, TERMINATION_DISABLED,
                                                    make_request_run, run_default_sc,
                                                    run_duchess, run_short_mk)
    from paper_2509_24957_b200.workload import SyntheticParams, generate_synthetic
    tr = trace("a", [tmpl(100, "a"), tmpl(200, "b"), tmpl(300, "a")])
    cfg = OrchestratorConfig(max_branches=3, interval_tokens=80)
    o = run_default_sc(tr, cfg)
    assert o.tokens_decode == 600 and o.final == "a" and o.termination_reason == "exhausted"
    with pytest.raises(ValueError, match="short_m"):
        make_request_run("short-mk", tr, OrchestratorConfig(max_branches=2, short_m=3))
    with pytest.raises(ValueError, match="dynasor_window"):
        DynasorRun(tr, OrchestratorConfig(dynasor_window=1))
    # crit 1: termination disabled + full fractions == plain self-consistency
    wl = generate_synthetic(SyntheticParams(templates_per_request=10), 12, seed=101)
    cfg = OrchestratorConfig(max_branches=10, interval_tokens=80,
                             early_term_threshold=TERMINATION_DISABLED, consensus_frac=1.0,
                             coverage_frac=1.0)
    for i, t in enumerate(wl.requests):
        sc = run_default_sc(t, cfg)
        du = run_duchess(t, cfg, random.Random(i))
        assert (du.tokens_total, du.tally, du.final) == (sc.tokens_total, sc.tally, sc.final)
    # crit 10: short-m@k == default SC at m = k; exactly m answers for m < k
    rng = random.Random(31)
    for trial in range(6):
        k = rng.randint(2, 10)
        t = trace("0", [tmpl(rng.randint(40, 500), str(rng.randint(0, 3))) for _ in range(k)])
        full = OrchestratorConfig(max_branches=k, interval_tokens=16, short_m=k)
        mk, sc = run_short_mk(t, full), run_default_sc(t, full)
        assert (mk.tally, mk.final, mk.tokens_total) == (sc.tally, sc.final, sc.tokens_total)
        m = rng.randint(1, k - 1)
        cut = run_short_mk(t, OrchestratorConfig(max_branches=k, interval_tokens=16, short_m=m))
        assert cut.tally.total == m
    run = DefaultScRun(tr, OrchestratorConfig(max_branches=3, interval_tokens=80))
    run.run()
    with pytest.raises(RuntimeError, match="request already terminated"):
        run.step()
    del CANCELLED


def test_dynasor_facade_probe_history_matches_oracle():
    """DynasorRun probes every active branch each round (orchestrator.py:539-556);
    the facade mirrors every probe into probe_history, as the oracle's
    DynasorRequest (and the reference) record them."""
    from oracle import port
    from paper_2509_24957_b200.orchestrator import DynasorRun, OrchestratorConfig
    from paper_2509_24957_b200.workload import SyntheticParams, generate_synthetic
    wl = generate_synthetic(SyntheticParams(templates_per_request=6), 6, seed=5)
    cfg = OrchestratorConfig(max_branches=4, interval_tokens=32, dynasor_window=3)
    knobs = port.Knobs(max_branches=4, interval_tokens=32, dynasor_window=3)
    for t in wl.requests:
        run = DynasorRun(t, cfg)
        run.run()
        ref = port.DynasorRequest(port.Trace(t.id, t.ground_truth, t.prompt_tokens,
                                             [port.Tmpl(x.natural_length, x.final_answer,
                                                        list(x.probes), x.oracle_convergence,
                                                        x.pred_probs) for x in t.templates],
                                             t.difficulty), knobs)
        ref.run()
        assert [b.probe_history for b in run.branches] == \
            [b.probe_history for b in ref.branches], t.id
        assert any(len(b.probe_history) > 1 for b in run.branches)
