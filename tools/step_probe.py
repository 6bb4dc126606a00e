"""Time the C2 step with and without per-K1 events (does event recording between
kernels cost overlap?)."""
import sys
import torch
sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2509_24957_b200 import _lib  # noqa: E402
from paper_2509_24957_b200.engine import BatchedDuchess  # noqa: E402
from paper_2509_24957_b200.probe import ProbeBank, Scorer, fill_windows  # noqa: E402
from paper_2509_24957_b200.scheduler import difficulty_queue  # noqa: E402

cfg = bench.CONFIGS["c2"]
traces, knobs, seeds = bench.make_workload(cfg, 1000)
eng = BatchedDuchess(traces, knobs, seeds, n_slots=cfg["R"], pred_source=_lib.PRED_DEVICE,
                     queue=difficulty_queue([t.difficulty for t in traces]), cycle=True)
w, b, g, beta = bench.make_probe(cfg["H"], 1)
sc = Scorer(ProbeBank.from_linear(w, b, g, beta), cfg["R"] * cfg["c"])
rows = cfg["R"] * cfg["c"]
slabs = [torch.empty((rows, 1, 32, 4096), dtype=torch.bfloat16, device="cuda") for _ in range(4)]
for i, s in enumerate(slabs):
    fill_windows(s, i)
logit = torch.empty((rows, 1), device="cuda")
probs = eng.probs.view(rows, 1)
eng.advance()
for mode in ("events", "noevents", "k1only", "roundonly", "events", "noevents"):
    for i in range(10):
        sc.score_list(slabs[i % 4], logit, probs, eng.t["active_rows"], eng.t["active_count"])
        eng.round()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 200
    e0.record()
    for i in range(n):
        if mode == "events":
            a, bb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
        if mode != "roundonly":
            sc.score_list(slabs[i % 4], logit, probs, eng.t["active_rows"], eng.t["active_count"])
        if mode == "events":
            bb.record()
        if mode != "k1only":
            eng.round()
    e1.record()
    torch.cuda.synchronize()
    print(mode, "us/step", round(e0.elapsed_time(e1) / n * 1e3, 1))
