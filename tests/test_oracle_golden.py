"""Pin the oracle restatement (oracle/port.py) to golden vectors produced by
running the reference itself (tests/golden/make_golden.py). CPU only."""

import random

import numpy as np
import pytest

from oracle import activations as oact
from oracle import port
from tests.golden_util import (STATUS, case_knobs, case_traces, fx, gen_params, load,
                               port_report_tuple, report_tuple, workload_digest)


@pytest.mark.parametrize("case", load("decisions.json"), ids=lambda c: c["name"])
def test_port_replays_reference_decisions(case):
    traces = case_traces(case)
    assert workload_digest(traces) == case["digest"]
    knobs = case_knobs(case)
    for trace, ref in zip(traces, case["requests"]):
        req = port.DuchessRequest(trace, knobs, random.Random(int(ref["seed"])), rho=case["rho"])
        reports = []
        while not req.done:
            reports.append(port_report_tuple(req.step()))
        assert reports == [report_tuple(r) for r in ref["reports"]]
        o = req.outcome
        assert (o.tally, o.final, o.termination_reason, o.tokens_decode, o.tokens_probe,
                o.rounds) == (ref["outcome"]["tally"], ref["outcome"]["final"],
                              ref["outcome"]["reason"], ref["outcome"]["tokens_decode"],
                              ref["outcome"]["tokens_probe"], ref["outcome"]["rounds"])
        got = [[b.status, b.final_answer, b.offset_base, b.tokens_decoded, b.streak,
                len(b.prediction_history), float(b.last_prediction).hex()] for b in req.branches]
        want = [[STATUS[s], fa, ob, td, st, npred, lp] for s, fa, ob, td, st, npred, lp
                in ref["branches"]]
        assert got == want


@pytest.mark.parametrize("case", load("baselines.json"), ids=lambda c: c["name"])
def test_port_replays_reference_baselines(case):
    traces = port.generate(gen_params(case["params"]), case["n"], case["workload_seed"])
    assert workload_digest(traces) == case["digest"]
    knobs = case_knobs(case)
    for trace, ref in zip(traces, case["requests"]):
        req = port.BASELINES[case["policy"]](trace, knobs)
        reports = []
        while not req.done:
            reports.append(port_report_tuple(req.step()))
        assert reports == [report_tuple(r) for r in ref["reports"]]
        o = req.outcome
        assert (o.tally, o.final, o.termination_reason, o.tokens_decode, o.tokens_probe,
                o.rounds) == tuple(ref["outcome"][k] for k in ("tally", "final", "reason",
                                                               "tokens_decode", "tokens_probe",
                                                               "rounds"))
        assert [[b.status, b.final_answer, b.offset_base, b.tokens_decoded]
                for b in req.branches] == [[STATUS[s], fa, ob, td] for s, fa, ob, td
                                           in ref["branches"]]


def test_port_decision_fixture_covers_every_path():
    seen_status, seen_reason, seen_kind = set(), set(), set()
    for case in load("decisions.json"):
        for r in case["requests"]:
            seen_reason.add(r["outcome"]["reason"])
            seen_status.update(b[0] for b in r["branches"])
            for rep in r["reports"]:
                seen_kind.update(a[0] for a in rep[5])
    assert seen_reason == {"consensus", "coverage", "exhausted"}
    assert seen_status == {1, 2, 3, 4}
    assert seen_kind == {1, 2, 3}


def test_port_branch_out_matches_reference():
    for case in load("primitives.json")["branch_out"]:
        probs = [fx(p) for p in case["probs"]]
        temp = fx(case["temperature"])
        assert [x.hex() for x in port.branch_out_weights(probs, temp)] == case["weights"]
        assert [port.branch_out_sample(probs, temp, random.Random(s))
                for s in range(8)] == case["draws"]
        rng = random.Random(case["seq_seed"])
        assert [port.branch_out_sample(probs, temp, rng) for _ in range(20)] == case["seq"]


def test_neumaier_restatement_equals_builtin_sum():
    rng = random.Random(5)
    for _ in range(2000):
        xs = [rng.random() ** rng.uniform(0.1, 8.0) for _ in range(rng.randint(1, 64))]
        assert port.neumaier_sum(xs) == sum(xs)
    assert port.neumaier_sum([0.1] * 10) == sum([0.1] * 10)


class _W:
    pass


def _mlp_from(case):
    w = _W()
    w.input_dim, w.layer_dims, w.head_dim = case["input_dim"], case["layer_dims"], case["head_dim"]
    w.activations = case["activations"]
    dims = [w.input_dim, *w.layer_dims, w.head_dim]
    w.weights = [np.array([fx(v) for v in m]).reshape(dims[k + 1], dims[k])
                 for k, m in enumerate(case["weights"])]
    w.biases = [np.array([fx(v) for v in b]) for b in case["biases"]]
    w.ln_gain = None if case["ln_gain"] is None else np.array([fx(v) for v in case["ln_gain"]])
    w.ln_bias = None if case["ln_bias"] is None else np.array([fx(v) for v in case["ln_bias"]])
    if case["bn"] is None:
        w.bn_mean = w.bn_var = w.bn_gain = w.bn_bias = None
    else:
        w.bn_mean, w.bn_var, w.bn_gain, w.bn_bias = [
            [np.array([fx(v) for v in vec]) for vec in part] for part in case["bn"]]
    return w


def test_port_mlp_forward_matches_reference():
    for case in load("primitives.json")["mlp"]:
        w = _mlp_from(case)
        logits, probs = port.mlp_forward(w, [fx(v) for v in case["x"]])
        np.testing.assert_allclose(logits, [fx(v) for v in case["logits"]], rtol=0, atol=1e-12)
        np.testing.assert_allclose(probs, [fx(v) for v in case["probs"]], rtol=0, atol=1e-12)


def test_pooled_probe_and_activation_regeneration():
    import hashlib
    for case in load("primitives.json")["pooled"]:
        win = oact.synth_window(*case["key"], case["T"], case["H"], case["bf16"])
        assert hashlib.sha256(win.tobytes()).hexdigest() == case["window_sha"]
        logit, prob = port.pooled_linear_probe(
            win, np.array([fx(v) for v in case["w"]]), fx(case["b"]),
            np.array([fx(v) for v in case["ln_gain"]]), np.array([fx(v) for v in case["ln_bias"]]))
        assert logit == pytest.approx(fx(case["logit"]), abs=1e-12)
        assert prob == pytest.approx(fx(case["prob"]), abs=1e-12)


def test_port_service_order_matches_next_request():
    for case in load("primitives.json")["orders"]:
        n = len(case["levels"])
        if case["policy"] == "fcfs":
            keys = [(case["arrivals"][j], j) for j in range(n)]
        else:
            keys = [(case["levels"][j], case["arrivals"][j], j) for j in range(n)]
        assert port.service_order(keys) == case["order"]


def test_port_confusion_sampling_matches_reference():
    for case in load("primitives.json")["confusion"]:
        rng = random.Random(case["seed"])
        assert [port.confused_level(case["level"], rng) for _ in range(50)] == case["seq"]


def test_port_generate_matches_reference():
    for case in load("primitives.json")["generate"]:
        traces = port.generate(gen_params(case["params"]), case["n"], case["seed"])
        assert workload_digest(traces) == case["digest"]


# Known-answer tests of the reference (test_orchestrator.py:41-126, test_core.py)
def test_reference_known_answers():
    assert port.branch_out_weights([0.8, 0.2], 1.0) == pytest.approx([0.8, 0.2])
    assert port.branch_out_weights([0.8, 0.2], 0.5) == pytest.approx([0.9412, 0.0588], abs=1e-4)
    assert port.request_termination({"a": 6}, 0.6, 0.8, 10) == "consensus"
    assert port.request_termination({"a": 4, "b": 4}, 0.6, 0.8, 10) == "coverage"
    assert port.request_termination({"a": 5, "b": 2}, 0.6, 0.8, 10) is None
    assert port.request_termination({"a": 8}, 0.6, 0.8, 10) == "consensus"
    assert port.majority_vote({"a": 1, "b": 1}) == "a"
    with pytest.raises(ValueError, match="no answers collected"):
        port.majority_vote({})
    with pytest.raises(ValueError, match="no branch to duplicate"):
        port.branch_out_weights([], 1.0)
