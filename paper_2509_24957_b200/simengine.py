"""Serving-timeline simulation over device round records (mirrors reference
simengine.py).

The reference runs one request at a time through ``make_request_run`` and
advances a clock round by round (simengine.py:150-281). Every request's
internal stream is seeded by workload order (simengine.py:191-193), so its
rounds never depend on the schedule or the clock. Here all requests run at
once in one batched device engine (``BatchedDuchess``, policy kernels of
decide.cu), and ``duchess_timeline`` folds each round record into a per-request
service time (sum of round_time + probe costs) and first-token offset on the
device. The host then replays only the single-server queue: arrivals,
prefills, the schedule's pick order and the clock, which are integer sums of
those per-request figures. Outputs (logs, metrics, CSV, JSON) are
byte-identical to the reference's for the same inputs.

Difficulty labels for ``easiest-predicted`` come from ``duchess_confused_levels``
(one draw per request from ``random.Random(predict_seeds[order])``,
simengine.py:223-227) or the trace label.
"""

from __future__ import annotations

import csv
import heapq
import json
import random
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from . import _lib
from .core import Duration, TimePoint, percentile
from .orchestrator import POLICIES, POLICY_DUCHESS, OrchestratorConfig
from .predictor import DEFAULT_CONFUSION, SyntheticPredictorConfig, validate_confusion
from .scheduler import EASIEST_ACTUAL, EASIEST_PREDICTED, FCFS, SCHEDULES
from .workload import Workload


@dataclass(frozen=True)
class TimingModel:
    """Linear-in-batch decode cost (simengine.py:27-48): a round of ``tokens``
    tokens over ``n`` branches costs tokens * (ms_per_token +
    ms_per_extra_branch * (n - 1)) ms; probes at the single-branch rate."""

    ms_per_token: float = 25.0
    ms_per_extra_branch: float = 0.0
    ms_per_prompt_token: float = 0.1

    def __post_init__(self) -> None:
        if self.ms_per_token <= 0:
            raise ValueError("ms_per_token must be > 0")
        if self.ms_per_extra_branch < 0:
            raise ValueError("ms_per_extra_branch must be >= 0")
        if self.ms_per_prompt_token < 0:
            raise ValueError("ms_per_prompt_token must be >= 0")


def round_time(active_branches: int, tokens: int, model: TimingModel) -> Duration:
    """Integer-ms wall time of one decode round (simengine.py:51-56); the
    device fold (duchess_timeline) evaluates the same double expression."""
    if active_branches < 1:
        raise ValueError("active_branches must be >= 1")
    per_token = model.ms_per_token + model.ms_per_extra_branch * (active_branches - 1)
    return int(round(tokens * per_token))


def prefill_time(prompt_tokens: int, model: TimingModel) -> Duration:
    return int(round(prompt_tokens * model.ms_per_prompt_token))


@dataclass
class RequestLogEntry:
    request_id: str
    arrival: TimePoint
    service_start: TimePoint
    first_token_time: TimePoint
    completion: TimePoint
    tokens_decode: int
    tokens_probe: int
    answers_collected: int
    final: str
    correct: bool
    termination_reason: str
    difficulty_actual: int | None
    difficulty_predicted: int | None

    @property
    def latency(self) -> Duration:
        return self.completion - self.arrival

    @property
    def ttft(self) -> Duration:
        return self.first_token_time - self.arrival




@dataclass
class MetricsReport:
    policy: str
    schedule: str
    n_requests: int
    accuracy: float
    latency_mean_ms: float
    latency_p50_ms: int
    latency_p95_ms: int
    ttft_mean_ms: float
    ttft_p50_ms: int
    ttft_p95_ms: int
    tokens_decode_mean: float
    tokens_total_mean: float
    seed: int
    workload_hash: str
    config: dict = field(default_factory=dict)

    def to_dict(self) -> dict:
        """Summary JSON layout (simengine.py:100-119)."""
        return {
            "policy": self.policy, "schedule": self.schedule, "n_requests": self.n_requests,
            "accuracy": self.accuracy,
            "latency_ms": {"mean": self.latency_mean_ms, "p50": self.latency_p50_ms,
                           "p95": self.latency_p95_ms},
            "ttft_ms": {"mean": self.ttft_mean_ms, "p50": self.ttft_p50_ms,
                        "p95": self.ttft_p95_ms},
            "tokens_per_request": {"decode_mean": self.tokens_decode_mean,
                                   "total_mean": self.tokens_total_mean},
            "seed": self.seed, "workload_hash": self.workload_hash, "config": self.config,
        }

    @classmethod
    def from_dict(cls, obj: dict) -> "MetricsReport":
        lat, ttft, tok = obj["latency_ms"], obj["ttft_ms"], obj["tokens_per_request"]
        return cls(policy=obj["policy"], schedule=obj["schedule"],
                   n_requests=obj["n_requests"], accuracy=obj["accuracy"],
                   latency_mean_ms=lat["mean"], latency_p50_ms=lat["p50"],
                   latency_p95_ms=lat["p95"], ttft_mean_ms=ttft["mean"],
                   ttft_p50_ms=ttft["p50"], ttft_p95_ms=ttft["p95"],
                   tokens_decode_mean=tok["decode_mean"], tokens_total_mean=tok["total_mean"],
                   seed=obj["seed"], workload_hash=obj["workload_hash"],
                   config=obj.get("config", {}))


class SimulationError(Exception):
    pass


# ---------------------------------------------------------------------------
# device part: every request's rounds, folded into service figures

@dataclass
class ServiceFigures:
    """Per request (workload order): decode-phase service time, first-token
    offset within it (-1 = no round decoded), and the outcome."""
    service_ms: np.ndarray
    first_token_ms: np.ndarray
    outcomes: list


def device_service(workload: Workload, config: OrchestratorConfig, policy: str,
                   policy_seeds: list, timing: TimingModel,
                   synthetic: SyntheticPredictorConfig, max_slots: int = 8192,
                   device="cuda") -> ServiceFigures:
    """Run every request of the workload through the device engine (all at
    once, up to max_slots concurrently) and fold its round records into
    service figures with duchess_timeline after every round."""
    import torch

    from .engine import BatchedDuchess
    _lib.require_cuda()
    lib = _lib.load()
    traces = workload.requests
    n = len(traces)
    eng = BatchedDuchess(traces, config, policy_seeds, n_slots=min(n, max_slots),
                         pred_source=_lib.PRED_TRACE, rho=synthetic.rho,
                         queue=list(range(n)), policy=policy, device=device)
    svc = torch.zeros(n, dtype=torch.int64, device=eng.device)
    first = torch.full((n,), -1, dtype=torch.int64, device=eng.device)
    probe_cost = round_time(1, config.probe_cost_tokens, timing)
    stream = _lib.stream_handle()
    duchess = policy == POLICY_DUCHESS
    if duchess:
        eng.advance()
    while True:
        for _ in range(8):                      # host checks completion every 8 rounds
            if duchess:
                eng.round()
            else:
                eng.baseline_round()
            _lib.check(lib.duchess_timeline(
                eng.t["round_rec"].data_ptr(), eng.R, float(timing.ms_per_token),
                float(timing.ms_per_extra_branch), int(probe_cost), svc.data_ptr(),
                first.data_ptr(), stream), "duchess_timeline")
        if eng.all_done():
            break
    outcomes = eng.outcomes()
    for o in outcomes:
        if o is None or o["error"]:
            raise ValueError("no answers collected")      # majority_vote, core.py:80-81
    return ServiceFigures(svc.cpu().numpy(), first.cpu().numpy(), outcomes)


def predicted_levels(workload: Workload, mode: str, predict_seeds: list, confusion,
                     device="cuda", weights=None, activations=None) -> list:
    """predict_difficulty(mode, ...) for every request with its own stream
    random.Random(predict_seeds[order]) (simengine.py:223-227). mode "mlp"
    (predictor.py:398-402: argmax of the complexity MLP + 1, which the
    reference's simulation rejects, simengine.py:184-186) runs the tensor-core
    classifier over every request's activation vector at once."""
    import torch

    from .engine import seed_states
    labels = [r.difficulty for r in workload.requests]
    if mode == "mlp":
        from .difficulty import TensorCoreClassifier
        X = np.asarray(activations, dtype=np.float64)
        if X.ndim != 2 or X.shape[0] != len(labels):
            raise ValueError("mlp mode needs one activation vector per request")
        return [int(v) for v in TensorCoreClassifier(weights, device=device).predict_levels(X)]
    if mode == "actual":
        for lv in labels:
            if lv is None:
                raise ValueError("actual mode requires a trace difficulty label")
        return list(labels)
    for lv in labels:
        if lv is None:
            raise ValueError("noisy-label mode requires a trace difficulty label")
    matrix = DEFAULT_CONFUSION if confusion is None else confusion
    validate_confusion(matrix)
    n = len(labels)
    _lib.require_cuda()
    lib = _lib.load()
    st = seed_states(predict_seeds, device=device)     # random.Random(seed), on the device
    lv = torch.tensor(labels, dtype=torch.int32, device=device)
    mat = torch.tensor(np.asarray(matrix, dtype=np.float64).reshape(-1), device=device)
    out = torch.empty(n, dtype=torch.int32, device=device)
    _lib.check(lib.duchess_confused_levels(st.data_ptr(), n, lv.data_ptr(), mat.data_ptr(),
                                           out.data_ptr(), _lib.stream_handle()),
               "duchess_confused_levels")
    return [int(v) for v in out.cpu().numpy()]


# ---------------------------------------------------------------------------
# host part: the single-server queue (simengine.py:196-270)

def run_simulation(workload: Workload, orch_config: OrchestratorConfig, policy: str,
                   schedule: str, arrivals: list, timing: TimingModel, seed: int,
                   synthetic: SyntheticPredictorConfig | None = None,
                   difficulty_mode: str | None = None,
                   confusion=None, difficulty_weights=None,
                   difficulty_activations=None) -> tuple:
    """One serving timeline over the whole workload (simengine.py:150-281).
    Returns (MetricsReport, [RequestLogEntry sorted by request id]).
    difficulty_mode "mlp" (an extension: the reference's simulation accepts
    only "actual" / "noisy-label") predicts levels with the complexity MLP
    `difficulty_weights` over `difficulty_activations` [n_requests, input_dim]
    (predict_difficulty("mlp"), predictor.py:398-402)."""
    if policy not in POLICIES:
        raise SimulationError(f"unknown policy {policy!r}")
    if schedule not in SCHEDULES:
        raise SimulationError(f"unknown schedule {schedule!r}")
    reqs = workload.requests
    if len(arrivals) != len(reqs):
        raise SimulationError(f"workload has {len(reqs)} requests but "
                              f"{len(arrivals)} arrivals supplied")
    if any(a > b for a, b in zip(arrivals, arrivals[1:])):
        raise SimulationError("arrivals must be sorted ascending")
    if schedule == EASIEST_ACTUAL:
        for r in reqs:
            if r.difficulty is None:
                raise SimulationError(f"request {r.id!r} has no difficulty label; "
                                      f"easiest-actual needs labeled traces")
    if schedule == EASIEST_PREDICTED:
        if difficulty_mode is None:
            raise SimulationError("easiest-predicted needs a difficulty predictor: pass "
                                  "difficulty_mode 'actual' or 'noisy-label'")
        if difficulty_mode not in ("actual", "noisy-label", "mlp"):
            raise SimulationError(
                f"unsupported difficulty mode {difficulty_mode!r} for simulation")
        if difficulty_mode == "mlp" and (difficulty_weights is None or
                                         difficulty_activations is None):
            raise SimulationError("mlp mode requires an activation vector and weights")
        if confusion is not None:
            validate_confusion(confusion)
    synthetic = synthetic or SyntheticPredictorConfig()

    master = random.Random(seed)                       # simengine.py:191-193
    policy_seeds = [master.getrandbits(64) for _ in reqs]
    predict_seeds = [master.getrandbits(64) for _ in reqs]

    fig = device_service(workload, orch_config, policy, policy_seeds, timing, synthetic)
    levels = (predicted_levels(workload, difficulty_mode, predict_seeds, confusion,
                               weights=difficulty_weights, activations=difficulty_activations)
              if schedule == EASIEST_PREDICTED else [None] * len(reqs))
    logs = replay_queue(workload, schedule, arrivals, timing, fig, levels)
    report = aggregate_metrics(logs, policy=policy, schedule=schedule, seed=seed,
                               workload_hash=workload.content_hash(),
                               config=_config_echo(orch_config, timing, synthetic,
                                                   difficulty_mode))
    return report, logs


def replay_queue(workload: Workload, schedule: str, arrivals: list, timing: TimingModel,
                 fig: ServiceFigures, levels: list) -> list:
    """The single-server queue of simengine.py:196-270 over precomputed
    per-request service figures; returns the logs sorted by request id."""
    reqs = workload.requests
    # arrival order (arrival, workload order); all admitted entries are
    # eligible at pick time (prefills run to completion first under
    # easiest-predicted), so the pick is a heap minimum on the schedule key
    by_arrival = sorted(range(len(reqs)), key=lambda i: (arrivals[i], i))

    def key(i):
        if schedule == FCFS:
            return (arrivals[i], i)
        if schedule == EASIEST_ACTUAL:
            return (reqs[i].difficulty, arrivals[i], i)
        return (levels[i], arrivals[i], i)

    heap: list = []
    prefill_queue: list = []       # easiest-predicted: admitted, not yet prefilled
    predicted: dict = {}
    clock, nxt = 0, 0
    logs = []

    def admit(now):
        nonlocal nxt
        while nxt < len(by_arrival) and arrivals[by_arrival[nxt]] <= now:
            i = by_arrival[nxt]
            nxt += 1
            if schedule == EASIEST_PREDICTED:
                heapq.heappush(prefill_queue, (arrivals[i], i))
            else:
                heapq.heappush(heap, (key(i), i))

    for _ in range(len(reqs)):
        admit(clock)
        if not heap and not prefill_queue:
            clock = arrivals[by_arrival[nxt]]
            admit(clock)
        if schedule == EASIEST_PREDICTED:            # run_prefills (:209-226)
            while True:
                admit(clock)
                if not prefill_queue:
                    break
                _, i = heapq.heappop(prefill_queue)
                clock += prefill_time(reqs[i].prompt_tokens, timing)
                predicted[i] = levels[i]
                heapq.heappush(heap, (key(i), i))
        _, i = heapq.heappop(heap)
        trace = reqs[i]
        service_start = clock
        if schedule != EASIEST_PREDICTED:
            clock += prefill_time(trace.prompt_tokens, timing)
        decode_start = clock
        clock = decode_start + int(fig.service_ms[i])
        ft = int(fig.first_token_ms[i])
        o = fig.outcomes[i]
        logs.append(RequestLogEntry(
            request_id=trace.id, arrival=arrivals[i], service_start=service_start,
            first_token_time=decode_start + ft if ft >= 0 else clock, completion=clock,
            tokens_decode=o["tokens_decode"], tokens_probe=o["tokens_probe"],
            answers_collected=sum(o["tally"].values()), final=o["final"],
            correct=o["final"] == trace.ground_truth, termination_reason=o["reason"],
            difficulty_actual=trace.difficulty, difficulty_predicted=predicted.get(i)))

    logs.sort(key=lambda e: e.request_id)
    return logs


def _config_echo(orch: OrchestratorConfig, timing: TimingModel,
                 synthetic: SyntheticPredictorConfig, difficulty_mode) -> dict:
    """Configuration echoed into the summary (simengine.py:284-313)."""
    knobs = ("max_branches", "interval_tokens", "early_term_threshold", "early_term_rounds",
             "branch_out_temperature", "consensus_frac", "coverage_frac", "token_cap",
             "probe_cost_tokens", "dynasor_window", "short_m")
    o = {k: getattr(orch, k) for k in knobs}
    if o["early_term_threshold"] == float("inf"):     # JSON has no infinity
        o["early_term_threshold"] = None
    echo = {"orchestrator": o,
            "timing": {"ms_per_token": timing.ms_per_token,
                       "ms_per_extra_branch": timing.ms_per_extra_branch,
                       "ms_per_prompt_token": timing.ms_per_prompt_token},
            "synthetic_rho": synthetic.rho}
    if difficulty_mode is not None:
        echo["difficulty_mode"] = difficulty_mode
    return echo


def aggregate_metrics(logs: list, *, policy: str, schedule: str, seed: int,
                      workload_hash: str, config: dict | None = None) -> MetricsReport:
    """simengine.py:316-339 (nearest-rank percentiles, plain means)."""
    if not logs:
        raise SimulationError("no log entries to aggregate")
    n = len(logs)
    lat = [e.latency for e in logs]
    ttft = [e.ttft for e in logs]
    return MetricsReport(
        policy=policy, schedule=schedule, n_requests=n,
        accuracy=sum(e.correct for e in logs) / n,
        latency_mean_ms=sum(lat) / n, latency_p50_ms=int(percentile(lat, 50)),
        latency_p95_ms=int(percentile(lat, 95)),
        ttft_mean_ms=sum(ttft) / n, ttft_p50_ms=int(percentile(ttft, 50)),
        ttft_p95_ms=int(percentile(ttft, 95)),
        tokens_decode_mean=sum(e.tokens_decode for e in logs) / n,
        tokens_total_mean=sum(e.tokens_decode + e.tokens_probe for e in logs) / n,
        seed=seed, workload_hash=workload_hash, config=config or {})


# ---------------------------------------------------------------------------
# stable output formats (simengine.py:345-372)

CSV_COLUMNS = ["request_id", "policy", "schedule", "arrival_ms", "service_start_ms",
               "first_token_ms", "completion_ms", "latency_ms", "ttft_ms", "tokens_decode",
               "tokens_probe", "answers", "correct", "termination_reason",
               "difficulty_actual", "difficulty_predicted"]


def _blank(v):
    return "" if v is None else v


def write_results_csv(logs: list, policy: str, schedule: str, path) -> None:
    with Path(path).open("w", encoding="utf-8", newline="") as fh:
        out = csv.writer(fh)
        out.writerow(CSV_COLUMNS)
        out.writerows([e.request_id, policy, schedule, e.arrival, e.service_start,
                       e.first_token_time, e.completion, e.latency, e.ttft, e.tokens_decode,
                       e.tokens_probe, e.answers_collected, "true" if e.correct else "false",
                       e.termination_reason, _blank(e.difficulty_actual),
                       _blank(e.difficulty_predicted)] for e in logs)


def write_summary_json(report_obj: dict, path) -> None:
    Path(path).write_text(json.dumps(report_obj, indent=2, sort_keys=True) + "\n",
                          encoding="utf-8")


# ---------------------------------------------------------------------------
# report comparison (simengine.py:375-433)

MATCHED_ACCURACY_TOLERANCE = 0.001      # within 0.1 percentage points

COMPARED_METRICS = [("latency_mean_ms", "latency mean"), ("latency_p50_ms", "latency p50"),
                    ("latency_p95_ms", "latency p95"), ("ttft_mean_ms", "ttft mean"),
                    ("ttft_p50_ms", "ttft p50"), ("ttft_p95_ms", "ttft p95"),
                    ("tokens_decode_mean", "tokens decode"),
                    ("tokens_total_mean", "tokens total"), ("accuracy", "accuracy")]


class ComparisonError(Exception):
    pass


def compare_reports(a: MetricsReport, b: MetricsReport) -> dict:
    """Signed relative deltas (b - a) / a in percent per metric."""
    if a.workload_hash != b.workload_hash:
        raise ComparisonError(f"reports cover different workloads: {a.workload_hash[:12]} vs "
                              f"{b.workload_hash[:12]}")
    rows = []
    for attr, label in COMPARED_METRICS:
        va, vb = getattr(a, attr), getattr(b, attr)
        rows.append({"metric": label, "a": va, "b": vb,
                     "delta_pct": None if va == 0 else (vb - va) / va * 100.0})
    side = lambda r: {"policy": r.policy, "schedule": r.schedule, "seed": r.seed}  # noqa: E731
    return {"a": side(a), "b": side(b), "workload_hash": a.workload_hash, "rows": rows,
            "matched_accuracy": abs(b.accuracy - a.accuracy) <= MATCHED_ACCURACY_TOLERANCE}


def format_comparison(comparison: dict) -> str:
    a, b = comparison["a"], comparison["b"]
    out = [f"a: {a['policy']}/{a['schedule']} (seed {a['seed']})",
           f"b: {b['policy']}/{b['schedule']} (seed {b['seed']})",
           f"{'metric':<16} {'a':>14} {'b':>14} {'delta':>10}"]
    for row in comparison["rows"]:
        d = "n/a" if row["delta_pct"] is None else f"{row['delta_pct']:+.1f}%"
        out.append(f"{row['metric']:<16} {row['a']:>14.4g} {row['b']:>14.4g} {d:>10}")
    if comparison["matched_accuracy"]:
        out.append("accuracy matched (|delta| <= 0.1 percentage points)")
    return "\n".join(out)
