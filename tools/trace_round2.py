"""Critical-path breakdown of the barrier-free round kernel at C2: for the
slowest slots, time per phase (globaltimer marks, relative to the earliest
slot start)."""
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
names = ["w123", "p23", "alive", "forks", "p5", "end", "clear+prologue", "phase1"]
agg = []
for step in range(60):
    sc.score_active(slab, logit, eng.probs.view(rows, 1), eng)
    torch.cuda.synchronize()
    tr.zero_()
    eng.round()
    torch.cuda.synchronize()
    if step < 20:
        continue
    t = tr.view(-1, 16).cpu().numpy().astype(np.float64)
    t0 = t[:, 12].min()
    live = t[:, 0] > 0
    rel = lambda k: (t[:, k] - t0) / 1e3  # noqa: E731
    marks = [rel(k) for k in (0, 1, 2, 3, 4, 5, 8, 10, 11)]
    endt = rel(11)
    worst = np.argsort(np.where(live, endt, -1))[-5:]
    for r in worst:
        ph = [marks[i + 1][r] - marks[i][r] for i in range(8)]
        agg.append(ph + [endt[r], rel(0)[r], t[r, 6], t[r, 7]])
a = np.array(agg)
print("slowest-slot phase medians (us):", {n: round(float(np.median(a[:, i])), 2) for i, n in enumerate(names)})
print("end median", np.median(a[:, 8]), "start (after wait) median", np.median(a[:, 9]),
      "forks med", np.median(a[:, 10]), "terms med", np.median(a[:, 11]))
