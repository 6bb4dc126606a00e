"""trace ingestion and answer interning, against fixtures made
by running the reference (tests/golden/make_golden.py ingestion): answer
normalisation (core.py:24-39), the JSONL schema v1 byte for byte plus the
content hash (workload.py:193-311; reference tests pkg/tests/test_workload.py
:74-84 pred_probs round trip, :129-139 generate -> save -> load round trip),
validate_trace violations (:114-191) and load_trace's error messages
(first defect in the reference's field order)."""

import json

import pytest

from paper_2509_24957_b200 import workload as W
from paper_2509_24957_b200.core import normalize_answer
from tests.golden_util import load

G = load("ingestion.json")


def with_pred_probs(requests, seed: int):
    """make_golden.py's helper: trace-embedded predictions on every other
    template, drawn from random.Random(seed)."""
    import random
    rng = random.Random(seed)
    out = []
    for r in requests:
        tmpls = []
        for j, t in enumerate(r.templates):
            pp = None
            if j % 2 == 0:
                ats = sorted(rng.sample(range(1, t.natural_length + 1), min(6, t.natural_length)))
                pp = [(a, round(rng.random(), 6)) for a in ats]
            tmpls.append(W.BranchTemplate(t.natural_length, t.final_answer, list(t.probes),
                                          t.oracle_convergence, pp))
        out.append(W.RequestTrace(r.id, r.ground_truth, r.prompt_tokens, tmpls, r.difficulty))
    return out


def test_normalize_answer_matches_reference():
    for raw, want in G["normalize"]:
        assert normalize_answer(raw) == want, raw
        assert normalize_answer(want) == want          # idempotent (core.py:27)


@pytest.mark.parametrize("case", G["jsonl"], ids=lambda c: c["name"])
def test_jsonl_bytes_and_hash_match_reference(case, tmp_path):
    from dataclasses import fields
    params = W.SyntheticParams(**{f.name: (tuple(case["params"][f.name])
                                           if isinstance(case["params"][f.name], list)
                                           else case["params"][f.name])
                                  for f in fields(W.SyntheticParams)})
    wl = W.generate_synthetic(params, case["n"], seed=case["seed"])
    if case["pred_probs_seed"] is not None:
        wl = W.Workload(with_pred_probs(wl.requests, case["pred_probs_seed"]))
    path = tmp_path / "w.jsonl"
    W.save_trace(wl, path)
    assert path.read_text() == case["bytes"]
    assert wl.content_hash() == case["hash"]
    # the reference's own file loads to the same workload and re-saves byte for byte
    ref = tmp_path / "ref.jsonl"
    ref.write_text(case["bytes"])
    loaded = W.load_trace(ref)
    assert loaded.content_hash() == case["loaded_hash"] == case["hash"]
    again = tmp_path / "again.jsonl"
    W.save_trace(loaded, again)
    assert again.read_bytes() == ref.read_bytes()


@pytest.mark.parametrize("case", G["load_errors"], ids=lambda c: c[0])
def test_load_trace_errors_match_reference(case, tmp_path):
    name, text, message = case
    path = tmp_path / f"{name}.jsonl"
    path.write_text(text + "\n")
    if message is None:
        W.load_trace(path)
        return
    with pytest.raises(W.TraceError) as exc:
        W.load_trace(path)
    assert str(exc.value) == message


@pytest.mark.parametrize("case", G["validate"], ids=lambda c: c[0])
def test_validate_trace_matches_reference(case):
    name, reqs, max_branches, want = case
    wl = W.Workload([W.RequestTrace(rid, gt, pt, [
        W.BranchTemplate(n, fa, [tuple(p) for p in probes], conv,
                         None if pp is None else [tuple(x) for x in pp])
        for n, fa, probes, conv, pp in tmpls], diff) for rid, gt, pt, diff, tmpls in reqs])
    got = [[v.level, v.where, v.message] for v in W.validate_trace(wl, max_branches=max_branches)]
    assert got == want


@pytest.mark.gpu
def test_trace_prediction_steps_match_reference():
    """The facade's trace_prediction runs the device lookup (no CPU path)."""
    t = W.BranchTemplate(100, "1", [], None, [(16, 0.25), (32, 0.75)])
    for pos, want in G["trace_prediction"]:
        assert W.trace_prediction(t, pos) == float.fromhex(want)


def test_pack_keys_order_like_tuples():
    """pack_keys sorts like (level, arrival, order[, tiebreak]) tuples on both
    the fixed-width fast path and the rank-packed path (scheduler.py:84-93)."""
    import random as _r

    import numpy as _np

    from paper_2509_24957_b200.scheduler import pack_keys
    rng = _r.Random(4)
    for wide in (False, True):
        for _ in range(20):
            n = rng.randint(1, 50)
            lv = [rng.choice([-2, 0, 7, 40]) if wide else rng.randint(0, 7) for _ in range(n)]
            ar = [rng.choice([0, 3, 2 ** 44]) if wide else rng.randint(0, 9) for _ in range(n)]
            od = [rng.randint(0, 5) for _ in range(n)]
            tb = list(range(n))
            keys = pack_keys(lv, ar, od, tiebreak=tb)
            got = [int(i) for i in _np.argsort(keys, kind="stable")]
            assert got == sorted(range(n), key=lambda j: (lv[j], ar[j], od[j], j))
            assert len(set(keys.tolist())) == n
