"""Sweep K1 launch configurations at the C2 shape (256 req x 16 branches x
T=32 x H=4096 bf16, 1 GiB per step), 4 rotating slabs (> L2), CUDA events."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2509_24957_b200.probe import ProbeBank, Scorer, fill_windows  # noqa: E402
import numpy as np  # noqa: E402

R, Cb, T, H, L = 256, 16, 32, 4096, 1
rows = R * Cb
rng = np.random.default_rng(0)
bank = ProbeBank.from_linear(rng.normal(0, 1.5 / 64, (1, H)), [0.0])
slabs = [torch.empty((rows, L, T, H), dtype=torch.bfloat16, device="cuda") for _ in range(4)]
for i, s in enumerate(slabs):
    fill_windows(s, 100 + i)
logit = torch.empty((rows, L), device="cuda")
prob = torch.empty((rows, L), dtype=torch.float64, device="cuda")
bytes_per_step = rows * L * T * H * 2
results = []
configs = [(0, 0), (1, 256), (1, 512), (2, 256), (2, 128), (4, 128), (4, 256), (8, 128), (2, 512)]
for ns, nt in configs:
    try:
        sc = Scorer(bank, rows * L, nsplit=ns, threads=nt)
        for i in range(5):
            sc(slabs[i % 4], logit, prob)
        torch.cuda.synchronize()
        n = 40
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for i in range(n):
            sc(slabs[i % 4], logit, prob)
        ev[1].record()
        torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1]) / n
        results.append({"nsplit": ns, "threads": nt, "us": ms * 1e3,
                        "GBps": bytes_per_step / (ms * 1e-3) / 1e9})
    except Exception as e:  # noqa: BLE001
        results.append({"nsplit": ns, "threads": nt, "error": str(e)})
    print(json.dumps(results[-1]), flush=True)
