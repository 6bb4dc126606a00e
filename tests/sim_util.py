"""Shared inputs for the simulation parity tests (tests/golden/simulation.json,
made by running the reference's run_simulation)."""

from __future__ import annotations

from oracle import port, simulate
from tests.golden_util import fx, gen_params, load


def cases():
    return load("simulation.json")


def facade_inputs(case):
    from paper_2509_24957_b200.orchestrator import OrchestratorConfig
    from paper_2509_24957_b200.predictor import SyntheticPredictorConfig
    from paper_2509_24957_b200.simengine import TimingModel
    from paper_2509_24957_b200.workload import SyntheticParams, generate_synthetic
    params = SyntheticParams(**{k: tuple(v) if isinstance(v, list) else v
                                for k, v in case["params"].items()})
    orch = dict(case["orchestrator"])
    orch["early_term_threshold"] = fx(orch["early_term_threshold"])
    workload = generate_synthetic(params, case["n"], seed=case["workload_seed"])
    return (workload, OrchestratorConfig(**orch), TimingModel(*case["timing"]),
            SyntheticPredictorConfig(rho=case["rho"]))


def oracle_traces_knobs(case):
    traces = port.generate(gen_params(case["params"]), case["n"], case["workload_seed"])
    orch = dict(case["orchestrator"])
    orch["early_term_threshold"] = fx(orch["early_term_threshold"])
    return traces, port.Knobs(**orch)


def oracle_figures(case):
    """Per-request (service_ms, first_token_offset, outcome dict) and
    predicted levels from the CPU oracle, in the product's ServiceFigures form."""
    import numpy as np

    from paper_2509_24957_b200.simengine import ServiceFigures
    traces, knobs = oracle_traces_knobs(case)
    ms_tok, extra, _ = case["timing"]
    pol, pred = simulate.seeds(len(traces), case["seed"])
    svc, first, outs = [], [], []
    for tr, s in zip(traces, pol):
        t, f, o = simulate.service(simulate.make_run(case["policy"], tr, knobs, s, case["rho"]),
                                   knobs, ms_tok, extra)
        svc.append(t)
        first.append(f)
        outs.append({"tokens_decode": o.tokens_decode, "tokens_probe": o.tokens_probe,
                     "tally": dict(o.tally), "final": o.final, "reason": o.termination_reason})
    levels = [None] * len(traces)
    if case["schedule"] == "easiest-predicted":
        import random
        if case["difficulty_mode"] == "actual":
            levels = [tr.difficulty for tr in traces]
        else:
            levels = [port.confused_level(tr.difficulty, random.Random(p),
                                          case["confusion"] or port.CONFUSION)
                      for tr, p in zip(traces, pred)]
    return ServiceFigures(np.array(svc), np.array(first), outs), levels
