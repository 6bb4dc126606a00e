"""Read-only stream rate vs working-set size (duchess_read_stream, CUDA events):
does a 64 GiB streaming pass (C5's per-GPU X) run slower than a 4 GiB one?"""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

dev = torch.device("cuda", 0)
for gib in (4, 16, 64):
    buf = torch.empty(gib << 30, dtype=torch.uint8, device=dev)
    buf.fill_(1)
    rates = [bench.measure_read_peak(dev, buf, reps=3) for _ in range(3)]
    print(f"{gib:3d} GiB: best {max(rates):.0f} GB/s, passes {[round(r) for r in rates]}", flush=True)
    del buf
    torch.cuda.empty_cache()
