"""Phase timing of the fused round kernel (duchess_step) at C2: per slot,
when its decision was claimed / started / ended relative to the kernel start,
and when the last window was scored (globaltimer marks)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2509_24957_b200 import _lib  # noqa: E402
from paper_2509_24957_b200.engine import BatchedDuchess  # noqa: E402
from paper_2509_24957_b200.probe import ProbeBank, fill_windows  # noqa: E402
from paper_2509_24957_b200.scheduler import difficulty_queue  # noqa: E402

import os
cfg = dict(bench.CONFIGS["c2"])
cfg["H"] = int(os.environ.get("TRACE_H", cfg["H"]))
cfg["T"] = int(os.environ.get("TRACE_T", cfg["T"]))
traces, knobs, seeds = bench.make_workload(cfg, 1000)
eng = BatchedDuchess(traces, knobs, seeds, n_slots=cfg["R"], pred_source=_lib.PRED_DEVICE,
                     queue=difficulty_queue([t.difficulty for t in traces]), cycle=True)
tr = eng.enable_trace()
w, b, g, beta = bench.make_probe(cfg["H"], 1)
bank = ProbeBank.from_linear(w, b, g, beta)
rows = cfg["R"] * cfg["c"]
slabs = [torch.empty((rows, 1, cfg["T"], cfg["H"]), dtype=torch.bfloat16, device="cuda")
         for _ in range(4)]
for i, s in enumerate(slabs):
    fill_windows(s, i)
logit = torch.empty(rows, device="cuda")
eng.begin_fused()
nodecide = len(sys.argv) > 1 and sys.argv[1] == "nodecide"
np.save("gpurun_out/trace_dummy.npy", np.zeros(1))
for step in range(40):
    if nodecide and step == 30:
        eng.policy.flags |= 2
    torch.cuda.synchronize()
    tr.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    eng.step_fused(slabs[step % 4], bank, logit)
    e1.record()
    torch.cuda.synchronize()
    if step >= 34:
        t = tr.view(-1, 16).cpu().numpy().astype(np.float64)
        np.save(f"gpurun_out/trace_step{step}{'_nd' if nodecide else ''}_H{cfg['H']}.npy", t)
        if nodecide:
            print(f"step {step}: event {e0.elapsed_time(e1)*1e3:.1f}us | stream end "
                  f"{(t[0,14]-t[0,13])/1e3:.1f}")
            continue
        t0 = t[0, 13]
        live = t[:, 12] > 0
        rel = lambda k: (t[live, k] - t0) / 1e3  # noqa: E731
        print(f"step {step}: event {e0.elapsed_time(e1)*1e3:.1f}us | stream end {(t[0,14]-t0)/1e3:.1f} "
              f"| claim max {rel(9).max():.1f} | decide start med {np.median(rel(12)):.1f} "
              f"p90 {np.percentile(rel(12), 90):.1f} max {rel(12).max():.1f} | decide end max "
              f"{rel(8).max():.1f} | p1 end max {rel(11).max():.1f} | decide dur med "
              f"{np.median(rel(8)-rel(12)):.2f} max {(rel(8)-rel(12)).max():.2f} | p1 dur med "
              f"{np.median(rel(11)-rel(8)):.2f} max {(rel(11)-rel(8)).max():.2f} | n {live.sum()}")
