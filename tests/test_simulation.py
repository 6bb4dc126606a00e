"""run_simulation parity (simengine.py:150-281).

CPU: the oracle's literal replay reproduces the reference's CSV bytes, and
the product's host-side queue replay + metrics + writers, fed the oracle's
per-request service figures, reproduce the reference's CSV and summary-JSON
bytes. GPU: the product's run_simulation (device engine + duchess_timeline)
reproduces both files byte for byte (criterion 9 of the reference's
acceptance suite: identical inputs -> identical output bytes)."""

import pytest

from oracle import simulate
from tests.sim_util import cases, facade_inputs, oracle_figures, oracle_traces_knobs

IDS = [c["name"] for c in cases()]


@pytest.mark.parametrize("case", cases(), ids=IDS)
def test_oracle_simulation_matches_reference_bytes(case):
    traces, knobs = oracle_traces_knobs(case)
    rows = simulate.simulate(traces, knobs, case["policy"], case["schedule"], case["arrivals"],
                             case["timing"], case["seed"], case["rho"],
                             case["difficulty_mode"], case["confusion"])
    assert simulate.csv_text(rows, case["policy"], case["schedule"]) == case["csv"]


def _write(tmp_path, logs, report, case):
    from paper_2509_24957_b200.simengine import write_results_csv, write_summary_json
    c, j = tmp_path / "r.csv", tmp_path / "r.json"
    write_results_csv(logs, case["policy"], case["schedule"], c)
    write_summary_json(report.to_dict(), j)
    return c.read_bytes().decode(), j.read_bytes().decode()


@pytest.mark.parametrize("case", cases(), ids=IDS)
def test_host_queue_replay_matches_reference_bytes(case, tmp_path):
    from paper_2509_24957_b200.simengine import _config_echo, aggregate_metrics, replay_queue
    workload, orch, timing, synth = facade_inputs(case)
    fig, levels = oracle_figures(case)
    logs = replay_queue(workload, case["schedule"], case["arrivals"], timing, fig, levels)
    report = aggregate_metrics(logs, policy=case["policy"], schedule=case["schedule"],
                               seed=case["seed"], workload_hash=workload.content_hash(),
                               config=_config_echo(orch, timing, synth, case["difficulty_mode"]))
    csv_text, json_text = _write(tmp_path, logs, report, case)
    assert csv_text == case["csv"]
    assert json_text == case["json"]


def test_round_time_known_answers():
    from paper_2509_24957_b200.simengine import TimingModel, round_time
    flat = TimingModel(ms_per_token=50.0, ms_per_extra_branch=0.0, ms_per_prompt_token=0.0)
    assert round_time(10, 16, flat) == 800                       # test_simengine.py:30-31
    assert round_time(10, 16, TimingModel(50.0, 5.0, 0.0)) == 1520
    assert round_time(1, 10, TimingModel(50.0, 5.0, 0.0)) == 500
    with pytest.raises(ValueError):
        round_time(0, 16, flat)


def test_simulation_input_validation():
    from paper_2509_24957_b200.orchestrator import OrchestratorConfig
    from paper_2509_24957_b200.simengine import SimulationError, TimingModel, run_simulation
    workload, orch, timing, _ = facade_inputs(cases()[0])
    arr = cases()[0]["arrivals"]
    with pytest.raises(SimulationError, match="unknown policy"):
        run_simulation(workload, orch, "nope", "fcfs", arr, timing, 0)
    with pytest.raises(SimulationError, match="unknown schedule"):
        run_simulation(workload, orch, "duchess", "nope", arr, timing, 0)
    with pytest.raises(SimulationError, match="arrivals supplied"):
        run_simulation(workload, orch, "duchess", "fcfs", arr[:-1], timing, 0)
    with pytest.raises(SimulationError, match="sorted ascending"):
        run_simulation(workload, orch, "duchess", "fcfs", arr[::-1], timing, 0)
    with pytest.raises(SimulationError, match="difficulty predictor"):
        run_simulation(workload, orch, "duchess", "easiest-predicted", arr, timing, 0)
    with pytest.raises(SimulationError, match="unsupported difficulty mode"):
        run_simulation(workload, orch, "duchess", "easiest-predicted", arr, timing, 0,
                       difficulty_mode="oracle")
    with pytest.raises(SimulationError, match="mlp mode requires"):
        run_simulation(workload, orch, "duchess", "easiest-predicted", arr, timing, 0,
                       difficulty_mode="mlp")
    assert isinstance(OrchestratorConfig(), OrchestratorConfig)
    assert TimingModel().ms_per_token == 25.0


@pytest.mark.gpu
@pytest.mark.parametrize("case", cases(), ids=IDS)
def test_device_run_simulation_matches_reference_bytes(case, tmp_path):
    from paper_2509_24957_b200.simengine import run_simulation
    workload, orch, timing, synth = facade_inputs(case)
    report, logs = run_simulation(workload, orch, case["policy"], case["schedule"],
                                  case["arrivals"], timing, case["seed"], synthetic=synth,
                                  difficulty_mode=case["difficulty_mode"],
                                  confusion=case["confusion"])
    csv_text, json_text = _write(tmp_path, logs, report, case)
    assert csv_text == case["csv"]
    assert json_text == case["json"]


@pytest.mark.gpu
def test_device_run_simulation_small_slot_pool(tmp_path):
    """Fewer device slots than requests (refills on device) gives the same bytes."""
    from paper_2509_24957_b200 import simengine
    case = cases()[0]
    workload, orch, timing, synth = facade_inputs(case)
    orig = simengine.device_service

    def few_slots(*a, **k):
        k["max_slots"] = 7
        return orig(*a, **k)
    simengine.device_service = few_slots
    try:
        report, logs = simengine.run_simulation(workload, orch, case["policy"], case["schedule"],
                                                case["arrivals"], timing, case["seed"],
                                                synthetic=synth)
    finally:
        simengine.device_service = orig
    assert _write(tmp_path, logs, report, case) == (case["csv"], case["json"])


@pytest.mark.gpu
@pytest.mark.parametrize("policy", ["duchess", "default-sc"])
def test_device_run_simulation_mlp_difficulty_matches_oracle(policy, tmp_path):
    """difficulty_mode="mlp" (the reference's simulation rejects
    it, simengine.py:184-186): levels from the tensor-core complexity MLP over
    per-request activations, the easiest-predicted queue and every byte of the
    CSV equal the oracle extension (oracle/simulate.py: fp64 mlp_forward
    argmax + 1 per request during its prefill, predictor.py:398-402)."""
    import numpy as np

    from oracle import simulate as osim
    from paper_2509_24957_b200.simengine import run_simulation
    from tests.test_gpu_difficulty import activations, complexity_mlp
    case = next(c for c in cases() if c["schedule"] == "easiest-predicted")
    workload, orch, timing, synth = facade_inputs(case)
    n = len(workload.requests)
    w = complexity_mlp(7, (512, 256, 256), head=5, act="gelu")
    X = activations(8, n, 512)
    report, logs = run_simulation(workload, orch, policy, "easiest-predicted", case["arrivals"],
                                  timing, case["seed"], synthetic=synth, difficulty_mode="mlp",
                                  difficulty_weights=w, difficulty_activations=X)
    traces, knobs = oracle_traces_knobs(case)
    rows = osim.simulate(traces, knobs, policy, "easiest-predicted",
                         case["arrivals"], case["timing"], case["seed"], case["rho"],
                         difficulty_mode="mlp", mlp_weights=w, mlp_activations=X)
    assert [(lg.request_id, lg.difficulty_predicted) for lg in logs] == \
        [(r[0], r[12]) for r in rows]
    assert len({r[12] for r in rows}) > 1
    c = tmp_path / "r.csv"
    from paper_2509_24957_b200.simengine import write_results_csv
    write_results_csv(logs, policy, "easiest-predicted", c)
    assert c.read_bytes().decode() == osim.csv_text(rows, policy, "easiest-predicted")
