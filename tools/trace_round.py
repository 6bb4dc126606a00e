"""Phase timing of the fused round kernel at C2 (globaltimer marks)."""
import sys
import numpy as np
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
tr = eng.enable_trace()
w, b, g, beta = bench.make_probe(cfg["H"], 1)
sc = Scorer(ProbeBank.from_linear(w, b, g, beta), cfg["R"] * cfg["c"])
rows = cfg["R"] * cfg["c"]
slab = torch.empty((rows, 1, 32, 4096), dtype=torch.bfloat16, device="cuda")
fill_windows(slab, 3)
logit = torch.empty((rows, 1), device="cuda")
eng.advance()
for step in range(40):
    sc.score_active(slab, logit, eng.probs.view(rows, 1), eng)
    torch.cuda.synchronize()
    tr.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    eng.round()
    e1.record()
    torch.cuda.synchronize()
    if step >= 35:
        t = tr.view(-1, 16).cpu().numpy().astype(np.float64)
        t0 = t[:, 12].min()
        rel = lambda k: (t[:, k] - t0) / 1e3  # noqa: E731
        np.save(f"gpurun_out/trace_round{step}.npy", t)
        print(f"step {step}: event {e0.elapsed_time(e1)*1e3:.1f}us | start max {rel(12).max():.2f} "
              f"decide_end max {rel(5).max():.2f} pre-sync max {rel(8).max():.2f} "
              f"post-sync min {rel(9).min():.2f} max {rel(9).max():.2f} prologue max {rel(10).max():.2f} "
              f"phase1 end max {rel(11).max():.2f} | median decide {np.median(rel(5)-rel(0)):.2f} "
              f"median prologue {np.median(rel(10)-rel(9)):.2f} median p1 {np.median(rel(11)-rel(10)):.2f}")
