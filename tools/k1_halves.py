"""Two half-size scorer launches PDL-chained on one stream vs one full launch
(same windows): does the second launch fill the first one's tail?"""
import sys
import torch
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
from paper_2509_24957_b200.probe import ProbeBank, Scorer, fill_windows  # noqa: E402

rows, T, H = 3724, 32, 4096
bank = ProbeBank.from_linear(np.random.default_rng(0).normal(0, 1 / 64, (1, H)), [0.0])
slabs = [torch.empty((rows, 1, T, H), dtype=torch.bfloat16, device="cuda") for _ in range(4)]
for i, s in enumerate(slabs):
    fill_windows(s, i)
sc = Scorer(bank, rows)
logit = torch.empty((rows, 1), device="cuda")
prob = torch.empty((rows, 1), dtype=torch.float64, device="cuda")
full = (torch.arange(rows, dtype=torch.int32, device="cuda"), torch.tensor([rows], dtype=torch.int32, device="cuda"))
h = rows // 2
half_a = (torch.arange(h, dtype=torch.int32, device="cuda"), torch.tensor([h], dtype=torch.int32, device="cuda"))
half_b = (torch.arange(h, rows, dtype=torch.int32, device="cuda"), torch.tensor([rows - h], dtype=torch.int32, device="cuda"))


def run(lists, n=100):
    for i in range(10):
        for lst, cnt in lists:
            sc.score_list(slabs[i % 4], logit, prob, lst, cnt)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(n):
        for lst, cnt in lists:
            sc.score_list(slabs[i % 4], logit, prob, lst, cnt)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


for _ in range(2):
    print(f"full {run([full]):.1f} us   two halves {run([half_a, half_b]):.1f} us   "
          f"four quarters {run([(torch.arange(q * rows // 4, (q + 1) * rows // 4, dtype=torch.int32, device='cuda'), torch.tensor([rows // 4], dtype=torch.int32, device='cuda')) for q in range(4)]):.1f} us")
