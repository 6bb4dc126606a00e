"""Critical-path breakdown of K2's barrier-free round kernel (duchess_round)
at C2 (one engine of R slots; the scorer runs and is synchronised first, so
the round kernel is timed alone): CUDA-event duration per launch, and per-slot
phase times from the kernel's globaltimer marks (DuchessState.trace):
w123 = state gather waves + scorer wait, p23 = predictions + early
termination, alive = alive list + raws, forks = branch-out loop + child
resolution, p5 = request termination + vote, end = outcome stores,
prologue = refill (atomic pop) or reload, phase1 = next round's phase 1,
exit = the list-parity exit counter (fence + atomic).

    python tools/trace_round.py [R] [config] [kv]

With `kv` each round is followed by its K3 update (duchess_kv_round) and the
K3 phases are reported: kv_forks (reset + forks), kv_release, kv_append.
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2509_24957_b200 import _lib  # noqa: E402
from paper_2509_24957_b200.engine import BatchedDuchess  # noqa: E402
from paper_2509_24957_b200.probe import ProbeBank, Scorer, fill_windows  # noqa: E402
from paper_2509_24957_b200.scheduler import difficulty_queue  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 128
name = sys.argv[2] if len(sys.argv) > 2 else "c2nokv"
use_kv = len(sys.argv) > 3 and sys.argv[3] == "kv"
cfg = dict(bench.CONFIGS[name], R=R)
traces, knobs, seeds = bench.make_workload(cfg, 1000)
eng = BatchedDuchess(traces, knobs, seeds, n_slots=R, pred_source=_lib.PRED_DEVICE,
                     queue=difficulty_queue([t.difficulty for t in traces]), cycle=True,
                     n_layers=cfg["L"], combine=1 if cfg["L"] > 1 else 0)
w, b, g, beta = bench.make_probe(cfg["H"], cfg["L"])
rows = R * cfg["c"]
sc = Scorer(ProbeBank.from_linear(w, b, g, beta), rows * cfg["L"])
slab = torch.empty((rows, cfg["L"], cfg["T"], cfg["H"]), dtype=torch.bfloat16, device="cuda")
fill_windows(slab, 3)
logit = torch.empty((rows, cfg["L"]), device="cuda")
eng.advance()
kv = None
if use_kv:
    from paper_2509_24957_b200.kvfork import PagedKVCache
    kv = PagedKVCache(eng, block_tokens=16, blocks_per_slot=4096, kv_bytes_per_token=4096)
    kv.round()
tr = None
names = ["w123", "p23", "alive", "forks", "p5", "end", "prologue", "phase1", "exit"]
agg, durs, allph, kvph, forkph = [], [], [], [], []
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for step in range(140):
    if step == 60:
        tr = eng.enable_trace()
    sc.score_active(slab, logit, eng.probs.view(rows, cfg["L"]), eng)
    torch.cuda.synchronize()
    if tr is not None:
        tr.zero_()
    ev0.record()
    eng.round()
    ev1.record()
    if kv is not None:
        kv.round()
    torch.cuda.synchronize()
    if step < 40:
        continue
    if tr is None:
        durs.append(ev0.elapsed_time(ev1) * 1e3)
        continue
    t = tr.view(-1, _lib.TRACE_WORDS).cpu().numpy().astype(np.float64)
    t0 = t[:, 12].min()
    live = t[:, 0] > 0
    rel = lambda k: (t[:, k] - t0) / 1e3  # noqa: E731
    marks = [rel(k) for k in (0, 1, 2, 3, 4, 5, 8, 10, 11, 13)]
    endt = rel(13)
    ph_all = np.stack([marks[i + 1] - marks[i] for i in range(9)], 1)[live]
    allph.append(ph_all)
    worst = np.argsort(np.where(live, endt, -1))[-5:]
    fr = live & (t[:, 20] > 0)
    forkph.append(np.stack([rel(20) - rel(3), rel(21) - rel(20), rel(22) - rel(21),
                            rel(4) - rel(22)], 1)[fr])
    if kv is not None:
        forked = live & (t[:, 17] > 0)         # decided, not reset (the fork / release phases)
        kvp = np.stack([rel(17) - rel(16), rel(18) - rel(17), rel(19) - rel(18),
                        rel(19) - rel(16)], 1)[forked]
        kvph.append(kvp)
    for r in worst:
        agg.append([marks[i + 1][r] - marks[i][r] for i in range(9)]
                   + [endt[r], rel(0)[r], t[r, 6], t[r, 7], endt[r] - rel(1)[r]])
a = np.array(agg)
ph = np.concatenate(allph)
print(f"config {name} R={R}: round kernel alone (events, untraced) median "
      f"{np.median(durs):.2f} us, min {np.min(durs):.2f}")
print("all-slot phase medians (us):",
      {n: round(float(np.median(ph[:, i])), 2) for i, n in enumerate(names)})
print("slowest-slot phase medians (us):",
      {n: round(float(np.median(a[:, i])), 2) for i, n in enumerate(names)})
print("slowest end (us from first start) median", round(float(np.median(a[:, 9])), 2),
      "| first mark after start median", round(float(np.median(a[:, 10])), 2),
      "| forks", float(np.median(a[:, 11])), "terms", float(np.median(a[:, 12])),
      "| after the scorer wait (the part not overlapped in the pipeline)",
      round(float(np.median(a[:, 13])), 2))
fk = np.concatenate(forkph) if forkph else None
if fk is not None and len(fk):
    print("fork sub-phases of slots that forked, median / p95 / max (us):",
          {n: (round(float(np.median(fk[:, i])), 2), round(float(np.percentile(fk[:, i], 95)), 2),
               round(float(fk[:, i].max()), 2))
           for i, n in enumerate(["setup (words, scans, draws)", "pick loop", "children",
                                  "stores"])})
if kvph:
    k = np.concatenate(kvph)
    print("K3 phases, all-slot median / p95 / max (us):",
          {n: (round(float(np.median(k[:, i])), 2), round(float(np.percentile(k[:, i], 95)), 2),
               round(float(k[:, i].max()), 2))
           for i, n in enumerate(["kv_forks", "kv_release", "kv_append", "kv_total"])})
