"""CPU restatement of the reference's serving simulation (simengine.py).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). A literal one-request-at-a-
time replay of simengine.py:150-281 over the oracle's request runs
(oracle/port.py), pinned to the reference's own CSV / summary-JSON bytes in
tests/golden/simulation.json. Also provides the per-request service figures
(decode-phase time, first-token offset, outcome) the GPU engine folds on the
device, so the product's host-side queue replay can be checked on CPU.
"""

from __future__ import annotations

import random

import numpy as np

from . import port


def round_time(n: int, tokens: int, ms_per_token: float, extra: float) -> int:
    """simengine.py:51-56."""
    if n < 1:
        raise ValueError("active_branches must be >= 1")
    return int(round(tokens * (ms_per_token + extra * (n - 1))))


def make_run(policy: str, trace, knobs, seed: int, rho: float):
    """orchestrator.py:564-577 make_request_run."""
    if policy == "duchess":
        return port.DuchessRequest(trace, knobs, random.Random(seed), rho=rho)
    return {"default-sc": port.DefaultScRequest, "short-mk": port.ShortMkRequest,
            "dynasor": port.DynasorRequest}[policy](trace, knobs)


def service(run, knobs, ms_per_token: float, extra: float):
    """simengine.py:244-257 inner loop, relative to the decode start:
    (service_ms, first_token_offset or -1, outcome)."""
    probe_cost = round_time(1, knobs.probe_cost_tokens, ms_per_token, extra)
    t, first = 0, -1
    while not run.done:
        rep = run.step()
        dt = 0
        if rep.decoding_branches > 0:
            dt += round_time(rep.decoding_branches, rep.max_chunk, ms_per_token, extra)
        dt += rep.probes * probe_cost
        t += dt
        if first < 0 and rep.decode_tokens > 0:
            first = t
    return t, first, run.outcome


def seeds(n: int, seed: int):
    """simengine.py:191-193: policy seeds, then predictor seeds."""
    master = random.Random(seed)
    pol = [master.getrandbits(64) for _ in range(n)]
    pred = [master.getrandbits(64) for _ in range(n)]
    return pol, pred


def simulate(traces, knobs, policy, schedule, arrivals, timing, seed, rho,
             difficulty_mode=None, confusion=None, mlp_weights=None, mlp_activations=None):
    """simengine.py:150-281 (validation omitted): log rows, one per request,
    sorted by request id: (id, arrival, start, first_token, completion,
    tokens_decode, tokens_probe, answers, final, correct, reason, actual,
    predicted)."""
    ms_tok, extra, ms_prompt = timing
    pol_seeds, pred_seeds = seeds(len(traces), seed)
    pending = sorted(range(len(traces)), key=lambda i: (arrivals[i], i))
    queue, logs = [], []
    prefilled, predicted = {}, {}
    clock, nxt = 0, 0

    def admit(now):
        nonlocal nxt
        while nxt < len(pending) and arrivals[pending[nxt]] <= now:
            queue.append(pending[nxt])
            nxt += 1

    def prefill(i):
        return int(round(traces[i].prompt_tokens * ms_prompt))

    while len(logs) < len(traces):
        admit(clock)
        if not queue:
            clock = arrivals[pending[nxt]]
            admit(clock)
        if schedule == "easiest-predicted":
            while True:                                      # run_prefills :209-226
                admit(clock)
                waiting = [i for i in queue if i not in prefilled]
                if not waiting:
                    break
                i = min(waiting, key=lambda j: (arrivals[j], j))
                clock += prefill(i)
                prefilled[i] = clock
                rng = random.Random(pred_seeds[i])
                if difficulty_mode == "actual":
                    predicted[i] = traces[i].difficulty
                elif difficulty_mode == "mlp":             # predictor.py:398-402
                    _z, probs = port.mlp_forward(mlp_weights, mlp_activations[i])
                    predicted[i] = int(np.argmax(probs)) + 1
                else:
                    predicted[i] = port.confused_level(traces[i].difficulty, rng,
                                                       confusion or port.CONFUSION)
        if schedule == "fcfs":
            keyf = lambda i: (arrivals[i], i)  # noqa: E731
        elif schedule == "easiest-actual":
            keyf = lambda i: (traces[i].difficulty, arrivals[i], i)  # noqa: E731
        else:
            keyf = lambda i: (predicted[i], arrivals[i], i)  # noqa: E731
        eligible = [i for i in queue if arrivals[i] <= clock and
                    (schedule != "easiest-predicted" or prefilled[i] <= clock)]
        i = min(eligible, key=keyf)
        queue.remove(i)
        start = clock
        if schedule != "easiest-predicted":
            clock += prefill(i)
        t0 = clock
        svc, first, out = service(make_run(policy, traces[i], knobs, pol_seeds[i], rho),
                                  knobs, ms_tok, extra)
        clock = t0 + svc
        tr = traces[i]
        logs.append((tr.id, arrivals[i], start, t0 + first if first >= 0 else clock, clock,
                     out.tokens_decode, out.tokens_probe, sum(out.tally.values()), out.final,
                     out.final == tr.ground_truth, out.termination_reason, tr.difficulty,
                     predicted.get(i)))
    logs.sort(key=lambda r: r[0])
    return logs


def csv_text(rows, policy: str, schedule: str) -> str:
    """simengine.py:352-365 layout (csv module, \\r\\n line ends)."""
    head = ("request_id,policy,schedule,arrival_ms,service_start_ms,first_token_ms,"
            "completion_ms,latency_ms,ttft_ms,tokens_decode,tokens_probe,answers,correct,"
            "termination_reason,difficulty_actual,difficulty_predicted")
    lines = [head]
    for (rid, arr, start, first, done, td, tp, ans, _final, ok, reason, act, pred) in rows:
        cells = [rid, policy, schedule, arr, start, first, done, done - arr, first - arr, td, tp,
                 ans, "true" if ok else "false", reason, "" if act is None else act,
                 "" if pred is None else pred]
        lines.append(",".join(str(c) for c in cells))
    return "\r\n".join(lines) + "\r\n"
