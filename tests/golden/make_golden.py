"""Generate golden fixtures by running the REFERENCE (/root/reference, read-only).

Run in the build container (the reference does not exist on the GPU box):
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py
The fixtures pin the oracle restatement (oracle/port.py, CPU tests) and the
CUDA path (GPU tests) to the reference's own outputs. Floats are stored as
float.hex() strings where bit-exactness matters.
"""

from __future__ import annotations

import hashlib
import json
import random
import sys
from dataclasses import replace
from pathlib import Path

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))

import numpy as np  # noqa: E402

from branchsim.orchestrator import (DefaultScRun, DuchessRun, DynasorRun,  # noqa: E402
                                    OrchestratorConfig, ShortMkRun,
                                    TERMINATION_DISABLED, branch_out_sample,
                                    branch_out_weights)
from branchsim.predictor import (DEFAULT_CONFUSION, SyntheticPredictorConfig,  # noqa: E402
                                 mlp_forward, sample_confused_level)
from branchsim.presets import PRESETS  # noqa: E402
from branchsim.scheduler import EASIEST_ACTUAL, FCFS, QueueEntry, next_request  # noqa: E402
from branchsim.workload import (BranchTemplate, RequestTrace,  # noqa: E402
                                SyntheticParams, generate_synthetic)
from util import random_mlp  # noqa: E402

OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(OUT.parent.parent))
from oracle import activations as oact  # noqa: E402

KIND = {"continue": 1, "terminate": 2, "branch_out": 3}
STATUS = {"active": 0, "early_terminated": 1, "natural_end": 2, "capped": 3, "cancelled": 4}


def workload_digest(requests) -> str:
    h = hashlib.sha256()
    for r in requests:
        h.update(json.dumps([r.id, r.ground_truth, r.prompt_tokens, r.difficulty,
                             [[t.natural_length, t.final_answer, [list(p) for p in t.probes],
                               t.oracle_convergence,
                               None if t.pred_probs is None else
                               [[a, float(p).hex()] for a, p in t.pred_probs]]
                              for t in r.templates]]).encode())
    return h.hexdigest()


def request_seeds(n: int, master_seed: int) -> list[int]:
    master = random.Random(master_seed)           # simengine.py:191-192
    return [master.getrandbits(64) for _ in range(n)]


def with_pred_probs(requests, seed: int):
    """Attach random trace-embedded predictions to every other template."""
    rng = random.Random(seed)
    out = []
    for r in requests:
        tmpls = []
        for j, t in enumerate(r.templates):
            pp = None
            if j % 2 == 0:
                ats = sorted(rng.sample(range(1, t.natural_length + 1),
                                        min(6, t.natural_length)))
                pp = [(a, round(rng.random(), 6)) for a in ats]
            tmpls.append(BranchTemplate(t.natural_length, t.final_answer, list(t.probes),
                                        t.oracle_convergence, pp))
        out.append(RequestTrace(r.id, r.ground_truth, r.prompt_tokens, tmpls, r.difficulty))
    return out


def trace_to_obj(r):
    return [r.id, r.ground_truth, r.prompt_tokens, r.difficulty,
            [[t.natural_length, t.final_answer, [list(p) for p in t.probes],
              t.oracle_convergence,
              None if t.pred_probs is None else [[a, float(p).hex()] for a, p in t.pred_probs]]
             for t in r.templates]]


def run_case(name, params, n, wseed, cfg, rho, master_seed, pred_seed=None, store_traces=False):
    requests = generate_synthetic(params, n, seed=wseed).requests
    if pred_seed is not None:
        requests = with_pred_probs(requests, pred_seed)
        store_traces = True
    seeds = request_seeds(n, master_seed)
    synth = SyntheticPredictorConfig(rho=rho)
    reqs = []
    for trace, seed in zip(requests, seeds):
        run = DuchessRun(trace, cfg, random.Random(seed), synthetic=synth)
        reports = []
        while not run.done:
            rep = run.step()
            reports.append([rep.round_index, rep.decoding_branches, rep.max_chunk,
                            rep.decode_tokens, rep.probes,
                            [[KIND[a.kind], a.branch_id,
                              -1 if a.source_branch_id is None else a.source_branch_id]
                             for a in rep.actions], int(rep.done)])
        o = run.outcome
        reqs.append({
            "seed": str(seed),
            "reports": reports,
            "outcome": {"tally": dict(sorted(o.tally.counts.items())), "final": o.final,
                        "reason": o.termination_reason, "tokens_decode": o.tokens_decode,
                        "tokens_probe": o.tokens_probe, "rounds": o.rounds},
            "branches": [[STATUS[b.status], b.final_answer, b.offset_base, b.tokens_decoded,
                          b.streak, len(b.prediction_history), float(b.last_prediction).hex()]
                         for b in run.branches],
        })
    case = {"name": name, "params": {k: getattr(params, k) for k in params.__dataclass_fields__},
            "n": n, "workload_seed": wseed, "master_seed": master_seed, "rho": rho,
            "config": {k: getattr(cfg, k) for k in cfg.__dataclass_fields__},
            "digest": workload_digest(requests), "requests": reqs}
    if store_traces:
        case["traces"] = [trace_to_obj(r) for r in requests]
    case["config"]["early_term_threshold"] = float(cfg.early_term_threshold).hex()
    return case


def decisions():
    gsm = PRESETS["gsm8k-like"]
    mmlu = PRESETS["mmlu-like"]
    math_ = PRESETS["math-like"]
    c1 = replace(gsm.orchestrator, max_branches=8)
    p64 = replace(gsm.synthetic, templates_per_request=64)
    cases = [
        run_case("c1_gsm8k_rho07", p64, 48, 7, c1, 0.7, 11),
        run_case("c1_gsm8k_rho1", p64, 32, 7, c1, 1.0, 11),
        run_case("lambda08", p64, 32, 8, replace(c1, branch_out_temperature=0.8), 0.6, 12),
        run_case("lambda03", p64, 24, 9, replace(c1, branch_out_temperature=0.3), 0.5, 13),
        run_case("capped", p64, 24, 10, replace(c1, token_cap=128), 0.6, 14),
        run_case("exhausted", replace(gsm.synthetic, templates_per_request=6), 24, 11,
                 replace(c1, consensus_frac=1.0, coverage_frac=1.0), 0.6, 15),
        run_case("no_terminate", replace(gsm.synthetic, templates_per_request=12), 16, 12,
                 replace(c1, early_term_threshold=TERMINATION_DISABLED, consensus_frac=1.0,
                         coverage_frac=1.0), 0.6, 16),
        run_case("pred_probs", p64, 24, 13, c1, 0.6, 17, pred_seed=99),
        run_case("mmlu", replace(mmlu.synthetic, templates_per_request=24), 24, 14,
                 mmlu.orchestrator, 0.7, 18),
        run_case("math_c16", replace(math_.synthetic, templates_per_request=64), 16, 15,
                 replace(math_.orchestrator, max_branches=16), 0.7, 19),
        run_case("wide_c48", replace(gsm.synthetic, templates_per_request=96), 8, 16,
                 replace(c1, max_branches=48, interval_tokens=32), 0.7, 20),
        run_case("c1_single", replace(gsm.synthetic, templates_per_request=3), 16, 17,
                 replace(c1, max_branches=1, early_term_rounds=1), 0.6, 21),
        # the device limit: 64 branch slots (both lane sets full), lambda 0.8 pow path
        run_case("max_c64", replace(gsm.synthetic, templates_per_request=160), 6, 18,
                 replace(c1, max_branches=64, interval_tokens=24, branch_out_temperature=0.8,
                         early_term_threshold=0.6, early_term_rounds=1), 0.6, 22),
    ]
    return cases


def run_baseline_case(name, policy, params, n, wseed, cfg):
    requests = generate_synthetic(params, n, seed=wseed).requests
    cls = {"default-sc": DefaultScRun, "short-mk": ShortMkRun, "dynasor": DynasorRun}[policy]
    reqs = []
    for trace in requests:
        run = cls(trace, cfg)
        reports = []
        while not run.done:
            rep = run.step()
            reports.append([rep.round_index, rep.decoding_branches, rep.max_chunk,
                            rep.decode_tokens, rep.probes,
                            [[KIND[a.kind], a.branch_id,
                              -1 if a.source_branch_id is None else a.source_branch_id]
                             for a in rep.actions], int(rep.done)])
        o = run.outcome
        reqs.append({"reports": reports,
                     "outcome": {"tally": dict(sorted(o.tally.counts.items())), "final": o.final,
                                 "reason": o.termination_reason,
                                 "tokens_decode": o.tokens_decode,
                                 "tokens_probe": o.tokens_probe, "rounds": o.rounds},
                     "branches": [[STATUS[b.status], b.final_answer, b.offset_base,
                                   b.tokens_decoded] for b in run.branches]})
    cfg_d = {k: getattr(cfg, k) for k in cfg.__dataclass_fields__}
    cfg_d["early_term_threshold"] = float(cfg.early_term_threshold).hex()
    return {"name": name, "policy": policy,
            "params": {k: getattr(params, k) for k in params.__dataclass_fields__},
            "n": n, "workload_seed": wseed, "config": cfg_d,
            "digest": workload_digest(requests), "requests": reqs}


def baselines():
    gsm = PRESETS["gsm8k-like"].synthetic
    math_ = PRESETS["math-like"]
    base = replace(math_.orchestrator, max_branches=10)
    return [
        run_baseline_case("sc_math", "default-sc", math_.synthetic, 20, 21, base),
        run_baseline_case("sc_capped", "default-sc", gsm, 20, 22,
                          replace(base, token_cap=160, interval_tokens=32)),
        run_baseline_case("sc_few_templates", "default-sc", replace(gsm, templates_per_request=6),
                          12, 23, base),
        run_baseline_case("mk_m5", "short-mk", math_.synthetic, 20, 24, replace(base, short_m=5)),
        run_baseline_case("mk_m1", "short-mk", gsm, 20, 25, replace(base, short_m=1,
                                                                      interval_tokens=16)),
        run_baseline_case("mk_mk", "short-mk", gsm, 12, 26, replace(base, short_m=10)),
        run_baseline_case("mk_capped", "short-mk", math_.synthetic, 16, 27,
                          replace(base, short_m=4, token_cap=320)),
        run_baseline_case("dyn_w3", "dynasor", math_.synthetic, 20, 28, base),
        run_baseline_case("dyn_w2", "dynasor", gsm, 20, 29, replace(base, dynasor_window=2,
                                                                      interval_tokens=16)),
        run_baseline_case("dyn_capped", "dynasor", math_.synthetic, 16, 30,
                          replace(base, dynasor_window=4, token_cap=400)),
    ]


def hexs(xs):
    return [float(x).hex() for x in xs]


def primitives():
    rng = random.Random(2024)
    bo = []
    temps = [1.0, 0.5, 0.8, 0.3, 2.5]
    for i in range(300):
        n = rng.randint(1, 16)
        probs = [rng.random() for _ in range(n)]
        if i % 7 == 0:
            probs[0] = 0.0
        if i % 11 == 0:
            probs[-1] = 1.0
        if i % 13 == 0:
            probs = [rng.random() * 1e-7 for _ in range(n)]
        temp = temps[i % len(temps)] if i % 3 else rng.uniform(0.2, 3.0)
        w = branch_out_weights(probs, temp)
        draws = [branch_out_sample(probs, temp, random.Random(s)) for s in range(8)]
        seq_rng = random.Random(1000 + i)
        seq = [branch_out_sample(probs, temp, seq_rng) for _ in range(20)]
        bo.append({"probs": hexs(probs), "temperature": float(temp).hex(), "weights": hexs(w),
                   "draws": draws, "seq_seed": 1000 + i, "seq": seq})

    mlps = []
    mrng = random.Random(77)
    for trial in range(40):
        head = 1 if trial % 2 == 0 else 5
        depth = trial % 4
        dims = [mrng.randint(4, 12) for _ in range(depth)]
        w = random_mlp(mrng, input_dim=mrng.randint(6, 16), layer_dims=dims, head_dim=head,
                       activation="relu" if trial % 3 else "gelu",
                       layernorm=trial % 5 != 0, batchnorm=trial % 2 == 1 and depth > 0)
        x = [mrng.uniform(-2.0, 2.0) for _ in range(w.input_dim)]
        logits, probs = mlp_forward(w, x)
        mlps.append({
            "input_dim": w.input_dim, "layer_dims": w.layer_dims, "head_dim": w.head_dim,
            "activations": w.activations,
            "weights": [hexs(m.reshape(-1)) for m in w.weights],
            "biases": [hexs(b) for b in w.biases],
            "ln_gain": None if w.ln_gain is None else hexs(w.ln_gain),
            "ln_bias": None if w.ln_bias is None else hexs(w.ln_bias),
            "bn": None if w.bn_mean is None else
            [[hexs(v) for v in part] for part in (w.bn_mean, w.bn_var, w.bn_gain, w.bn_bias)],
            "x": hexs(x), "logits": hexs(logits), "probs": hexs(probs)})

    # pooled-window probe: reference mlp_forward on the fp64 mean of the stored
    # bf16 windows (the restated pooling + the reference's own forward)
    pooled = []
    prng = np.random.default_rng(5)
    for k in range(6):
        H, T = 256, (1, 4, 32)[k % 3]
        w = prng.normal(0, 1.5 / np.sqrt(H), size=(1, H))
        from branchsim.predictor import MlpWeights
        mw = MlpWeights(input_dim=H, layer_dims=[], head_dim=1, activations=[],
                        weights=[w], biases=[np.array([0.1 * k])],
                        ln_gain=prng.uniform(0.5, 1.5, H), ln_bias=prng.uniform(-0.1, 0.1, H))
        key = (1, 100 + k, k % 3, 16 * (k + 1), 0)
        win = oact.synth_window(*key, T, H, bf16=k % 2 == 0)
        logits, probs = mlp_forward(mw, win.astype(np.float64).mean(axis=0))
        pooled.append({"key": key, "T": T, "H": H, "bf16": k % 2 == 0, "w": hexs(w[0]),
                       "b": float(0.1 * k).hex(), "ln_gain": hexs(mw.ln_gain),
                       "ln_bias": hexs(mw.ln_bias), "logit": float(logits[0]).hex(),
                       "prob": float(probs[0]).hex(),
                       "window_sha": hashlib.sha256(win.tobytes()).hexdigest()})

    orders = []
    orng = random.Random(31)
    for i in range(60):
        n = orng.randint(1, 40)
        levels = [orng.randint(1, 5) for _ in range(n)]
        arrivals = sorted(orng.sample(range(0, 10 * n + 10), n))
        traces = [RequestTrace(f"q{j}", "1", 0, [BranchTemplate(10, "1")], levels[j])
                  for j in range(n)]
        perm = list(range(n))
        orng.shuffle(perm)
        for policy in (FCFS, EASIEST_ACTUAL):
            queue = [QueueEntry(traces[j], arrivals[j], j) for j in perm]
            got = []
            while queue:
                got.append(next_request(queue, policy, 10 ** 9).order)
            orders.append({"levels": levels, "arrivals": arrivals, "insert": perm,
                           "policy": policy, "order": got})

    conf = []
    for s in range(20):
        r = random.Random(500 + s)
        conf.append({"seed": 500 + s, "level": 1 + s % 5,
                     "seq": [sample_confused_level(1 + s % 5, DEFAULT_CONFUSION, r)
                             for _ in range(50)]})

    gens = []
    for name, params, n, seed in [("default", SyntheticParams(), 20, 1),
                                  ("gsm64", replace(PRESETS["gsm8k-like"].synthetic,
                                                    templates_per_request=64), 12, 7),
                                  ("math", PRESETS["math-like"].synthetic, 15, 3),
                                  ("mix", replace(SyntheticParams(),
                                                  level_mix=(1, 2, 3, 2, 1)), 10, 5)]:
        reqs = generate_synthetic(params, n, seed).requests
        gens.append({"name": name, "params": {k: getattr(params, k)
                                              for k in params.__dataclass_fields__},
                     "n": n, "seed": seed, "digest": workload_digest(reqs)})
    return {"branch_out": bo, "mlp": mlps, "pooled": pooled, "orders": orders,
            "confusion": conf, "generate": gens}


def simulation():
    """run_simulation (simengine.py:150-281) outputs: the exact CSV and
    summary-JSON bytes the reference writes, per case."""
    import dataclasses
    import dataclasses
    import tempfile

    from branchsim.presets import PRESETS as P
    from branchsim.scheduler import ArrivalConfig, gen_arrivals
    from branchsim.simengine import (TimingModel, run_simulation, write_results_csv,
                                     write_summary_json)
    cases = []
    specs = [
        # name, preset, n, wseed, orch overrides, policy, schedule, qpm, aseed, timing, seed,
        # rho, difficulty_mode, confusion
        ("fcfs_duchess", "gsm8k-like", 40, 5, {}, "duchess", "fcfs", 3.0, 1,
         (25.0, 0.0, 0.1), 9, 0.8, None, None),
        ("actual_default_sc", "gsm8k-like", 30, 6, {}, "default-sc", "easiest-actual", 2.0, 2,
         (25.0, 1.5, 0.2), 3, 0.8, None, None),
        ("predicted_noisy_duchess", "math-like", 30, 7, {}, "duchess", "easiest-predicted",
         4.0, 3, (20.0, 2.0, 0.3), 11, 0.7, "noisy-label", None),
        ("predicted_actual_short_mk", "mmlu-like", 25, 8, {"short_m": 4}, "short-mk",
         "easiest-predicted", 2.5, 4, (25.0, 0.5, 0.1), 5, 0.8, "actual", None),
        ("fcfs_dynasor", "math-like", 25, 9, {"dynasor_window": 2}, "dynasor", "fcfs", 1.0, 5,
         (30.0, 0.0, 0.0), 2, 0.8, None, None),
        ("predicted_confusion_duchess", "gsm8k-like", 35, 10,
         {"early_term_threshold": float("inf")}, "duchess", "easiest-predicted", 6.0, 6,
         (25.0, 0.25, 0.1), 17, 0.9, "noisy-label",
         [[0.5, 0.2, 0.1, 0.1, 0.1], [0.1, 0.5, 0.2, 0.1, 0.1], [0.1, 0.1, 0.5, 0.2, 0.1],
          [0.1, 0.1, 0.1, 0.5, 0.2], [0.2, 0.1, 0.1, 0.1, 0.5]]),
        ("burst_fcfs_duchess_lambda", "math-like", 30, 12, {"branch_out_temperature": 0.5,
                                                            "max_branches": 6},
         "duchess", "fcfs", 60.0, 7, (25.0, 3.0, 0.5), 23, 0.6, None, None),
    ]
    with tempfile.TemporaryDirectory() as tmp:
        for (name, preset, n, wseed, over, policy, schedule, qpm, aseed, tm, seed, rho, dmode,
             conf) in specs:
            params = P[preset].synthetic
            orch = dataclasses.replace(P[preset].orchestrator, **over)
            workload = generate_synthetic(params, n, seed=wseed)
            arrivals = gen_arrivals(ArrivalConfig(rate_qpm=qpm, n_requests=n, seed=aseed))
            timing = TimingModel(*tm)
            report, logs = run_simulation(workload, orch, policy, schedule, arrivals, timing,
                                          seed, synthetic=SyntheticPredictorConfig(rho=rho),
                                          difficulty_mode=dmode, confusion=conf)
            cpath, jpath = Path(tmp) / "r.csv", Path(tmp) / "r.json"
            write_results_csv(logs, policy, schedule, cpath)
            write_summary_json(report.to_dict(), jpath)
            orch_d = dataclasses.asdict(orch)
            orch_d["early_term_threshold"] = float(orch_d["early_term_threshold"]).hex()
            cases.append({"name": name, "params": dataclasses.asdict(params), "n": n,
                          "workload_seed": wseed, "orchestrator": orch_d, "policy": policy,
                          "schedule": schedule, "qpm": qpm, "arrival_seed": aseed,
                          "arrivals": arrivals, "timing": list(tm), "seed": seed, "rho": rho,
                          "difficulty_mode": dmode, "confusion": conf,
                          "csv": cpath.read_bytes().decode(), "json": jpath.read_bytes().decode()})
    return cases


def ingestion():
    """(f)2: answer normalisation, the JSONL schema (bytes + content hash),
    validate_trace violations and load_trace error messages of the reference
    (core.py:24-39, workload.py:114-311)."""
    import dataclasses
    import tempfile

    from branchsim.core import normalize_answer
    from branchsim.workload import (TraceError, Workload, load_trace, save_trace,
                                    trace_prediction, validate_trace)
    raws = ["42", "  42 ", "\\boxed{42}", "\\boxed{ {X} }", "{{7}}", "{}", "", "   ",
            "\\boxed{}", "ABC", "ǅemal", "{\\boxed{Yes}}", "\\boxed{a}b}", "{ 1/2 }",
            "STRASSE", "İstanbul", "{\\boxed{{3.0}}}", "\\boxed{x", "x}", "{ }"]
    out = {"normalize": [[r, normalize_answer(r)] for r in raws]}
    out["jsonl"] = []
    with tempfile.TemporaryDirectory() as d:
        for name, params, n, seed in [("default", SyntheticParams(), 12, 4),
                                      ("math", replace(PRESETS["math-like"].synthetic,
                                                       templates_per_request=9), 7, 21)]:
            w = generate_synthetic(params, n, seed=seed)
            w = Workload(with_pred_probs(w.requests, seed)) if name == "math" else w
            path = Path(d) / f"{name}.jsonl"
            save_trace(w, path)
            loaded = load_trace(path)
            out["jsonl"].append({"name": name, "params": dataclasses.asdict(params), "n": n,
                                 "seed": seed, "pred_probs_seed": seed if name == "math" else None,
                                 "bytes": path.read_bytes().decode(),
                                 "hash": w.content_hash(), "loaded_hash": loaded.content_hash()})
        bad = []
        good = {"v": 1, "id": "r0", "ground_truth": "42", "prompt_tokens": 10,
                "branches": [{"natural_length": 100, "final_answer": "42",
                              "probes": [{"at": 16, "answer": "7"}]}]}
        def variant(**kw):
            o = json.loads(json.dumps(good))
            for k, v in kw.items():
                if v is None:
                    o.pop(k, None)
                else:
                    o[k] = v
            return json.dumps(o)
        cases = {
            "missing_gt": variant(ground_truth=None),
            "missing_id_and_gt": variant(id=None, ground_truth=None),
            "bad_pt_and_branches": variant(prompt_tokens="x", branches=None),
            "bool_pt": variant(prompt_tokens=True),
            "bad_version": variant(v=2),
            "bad_difficulty": variant(difficulty="hard"),
            "bad_branch": variant(branches=[3]),
            "branch_missing_fields": variant(branches=[{"probes": [{"at": "x"}]}]),
            "bad_pred": variant(branches=[{"natural_length": 10, "final_answer": "1",
                                           "pred_probs": [{"at": 1, "p": "hi"}]}]),
            "probe_order": variant(branches=[{"natural_length": 100, "final_answer": "1",
                                              "probes": [{"at": 20, "answer": "1"},
                                                         {"at": 10, "answer": "2"}]}]),
            "empty_gt": variant(ground_truth=" {} "),
            "not_object": "[1, 2]",
            "malformed": "{\"v\": 1,",
            "duplicate": variant() + "\n" + variant(),
        }
        for name, text in cases.items():
            path = Path(d) / f"bad_{name}.jsonl"
            path.write_text(text + "\n")
            try:
                load_trace(path)
                bad.append([name, text, None])
            except TraceError as exc:
                bad.append([name, text, str(exc)])
        out["load_errors"] = bad
    tv = []
    mk = lambda n, fa, probes=(), conv=None, pp=None: BranchTemplate(n, fa, list(probes), conv, pp)
    vcases = [
        ("clean", [RequestTrace("a", "1", 5, [mk(100, "1")], 2)], None),
        ("degraded", [RequestTrace("a", "1", 5, [mk(100, "1")], None)], 4),
        ("empty_gt", [RequestTrace("a", "", 5, [mk(100, "1")], None)], None),
        ("probe_beyond_conv", [RequestTrace("a", "42", 0, [mk(100, "42", [(95, "7")], 90)],
                                            None)], None),
        ("many", [RequestTrace("a", "1", -1, [], 9),
                  RequestTrace("a", "1", 3, [mk(0, "1", [(5, "2"), (3, "1")], 200,
                                                 [(3, 0.5), (2, 1.5)])], None)], 2),
    ]
    for name, reqs, mb in vcases:
        vs = validate_trace(Workload(reqs), max_branches=mb)
        tv.append([name, [[r.id, r.ground_truth, r.prompt_tokens, r.difficulty,
                           [[t.natural_length, t.final_answer, [list(p) for p in t.probes],
                             t.oracle_convergence,
                             None if t.pred_probs is None else [list(x) for x in t.pred_probs]]
                            for t in r.templates]] for r in reqs],
                   mb, [[v.level, v.where, v.message] for v in vs]])
    out["validate"] = tv
    tp = mk(100, "1", pp=[(16, 0.25), (32, 0.75)])
    out["trace_prediction"] = [[x, trace_prediction(tp, x).hex()] for x in (0, 10, 16, 20, 32, 99)]
    return out


def main():
    (OUT / "ingestion.json").write_text(json.dumps(ingestion(), separators=(",", ":")))
    (OUT / "decisions.json").write_text(json.dumps(decisions(), separators=(",", ":")))
    (OUT / "baselines.json").write_text(json.dumps(baselines(), separators=(",", ":")))
    (OUT / "primitives.json").write_text(json.dumps(primitives(), separators=(",", ":")))
    (OUT / "simulation.json").write_text(json.dumps(simulation(), separators=(",", ":")))
    for p in sorted(OUT.glob("*.json")):
        print(p.name, p.stat().st_size)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "ingestion":
        (OUT / "ingestion.json").write_text(json.dumps(ingestion(), separators=(",", ":")))
    elif len(sys.argv) > 1 and sys.argv[1] == "simulation":
        (OUT / "simulation.json").write_text(json.dumps(simulation(), separators=(",", ":")))
    elif len(sys.argv) > 1 and sys.argv[1] == "decisions":
        (OUT / "decisions.json").write_text(json.dumps(decisions(), separators=(",", ":")))
    else:
        main()
