"""Per-slot decide phase timing at the C2 bench workload (globaltimer)."""
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
q = difficulty_queue([t.difficulty for t in traces])
eng = BatchedDuchess(traces, knobs, seeds, n_slots=cfg["R"], pred_source=_lib.PRED_DEVICE, queue=q, cycle=True)
tr = eng.enable_trace()
w, b, g, beta = bench.make_probe(cfg["H"], 1)
bank = ProbeBank.from_linear(w, b, g, beta)
sc = Scorer(bank, cfg["R"] * cfg["c"])
rows = cfg["R"] * cfg["c"]
slab = torch.empty((rows, 1, cfg["T"], cfg["H"]), dtype=torch.bfloat16, device="cuda")
fill_windows(slab, 5)
logit = torch.empty((rows, 1), device="cuda")
eng.advance()
for step in range(40):
    sc.score_active(slab, logit, eng.probs.view(rows, 1), eng)
    tr.zero_()
    eng.decide()
    torch.cuda.synchronize()
    if step >= 30:
        t = tr.view(-1, 8).cpu().numpy()
        live = t[:, 0] > 0
        t0 = t[live, 0].min()
        rel = (t[live, :6] - t0) / 1e3
        dur = rel[:, 5] - rel[:, 0]
        order = np.argsort(-dur)[:5]
        print(f"step {step}: slots={live.sum()} start_spread={rel[:,0].max():.1f}us "
              f"end_max={rel[:,5].max():.1f}us median_dur={np.median(dur):.2f}us")
        for i in order:
            ph = np.diff(rel[i])
            print(f"   slot dur={dur[i]:6.2f}us start={rel[i,0]:5.1f} phases(load,p23,p4a,forks,p5)={np.round(ph,2)} forks={t[live][i,6]} term={t[live][i,7]}")
    eng.advance()
