"""Time the C2 round back to back (no events between launches) for the
fused step (duchess_step), the fused step with decisions switched off
(scoring only, same launch shape), the split pair (K1 + duchess_round), K1
alone and the round kernel alone."""
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
w, b, g, beta = bench.make_probe(cfg["H"], 1)
bank = ProbeBank.from_linear(w, b, g, beta)
rows = cfg["R"] * cfg["c"]
slabs = [torch.empty((rows, 1, 32, 4096), dtype=torch.bfloat16, device="cuda") for _ in range(4)]
for i, s in enumerate(slabs):
    fill_windows(s, i)
logit = torch.empty((rows, 1), device="cuda")


def engine():
    return BatchedDuchess(traces, knobs, seeds, n_slots=cfg["R"], pred_source=_lib.PRED_DEVICE,
                          queue=difficulty_queue([t.difficulty for t in traces]), cycle=True)


def timeit(fn, n=200):
    for i in range(20):
        fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(n):
        fn(i)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


modes = sys.argv[1:] or ["fused", "nodecide", "split", "k1only", "roundonly", "fused"]
for mode in (modes if __name__ == "__main__" else []):
    eng = engine()
    sc = Scorer(bank, rows)
    probs = eng.probs.view(rows, 1)
    if mode in ("fused", "nodecide"):
        eng.begin_fused()
        for i in range(20):
            eng.step_fused(slabs[i % 4], bank, logit.view(-1))
        if mode == "nodecide":
            eng.policy.flags |= _lib.FLAG_PROFILE_NO_DECIDE
        us = timeit(lambda i: eng.step_fused(slabs[i % 4], bank, logit.view(-1)))
    else:
        eng.advance()
        for i in range(20):
            sc.score_active(slabs[i % 4], logit, probs, eng)
            eng.round()

        def f(i):
            if mode != "roundonly":
                sc.score_active(slabs[i % 4], logit, probs, eng)
            if mode != "k1only":
                eng.round()
        us = timeit(f)
    print(f"{mode:10s} us/step {us:.1f}", flush=True)
