"""Short-window K1 (T*H*esz <= 16 KB) timing: score_list over R*C windows of
T=1, H=5120, L=4 bf16 (C3-T1) and T=1, H=4096 fp32 (C1), best of 20."""
import sys
import torch
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
from paper_2509_24957_b200.probe import ProbeBank, Scorer, fill_windows  # noqa: E402

CASES = [(16384, 4, 1, 5120, torch.bfloat16), (4096, 1, 1, 4096, torch.float32),
         (64, 1, 1, 4096, torch.float32), (4096, 1, 32, 4096, torch.bfloat16),
         (65536, 4, 1, 5120, torch.bfloat16), (65536, 1, 1, 4096, torch.bfloat16)]
for rows, L, T, H, dt in [CASES[int(i)] for i in sys.argv[1:]] or CASES:
    rng = np.random.default_rng(0)
    bank = ProbeBank.from_linear(rng.normal(0, 0.02, (L, H)), np.zeros(L))
    slabs = [torch.empty((rows, L, T, H), dtype=dt, device="cuda") for _ in range(3)]
    for i, a in enumerate(slabs):
        fill_windows(a, i)
    lst = torch.arange(rows, dtype=torch.int32, device="cuda")
    cnt = torch.tensor([rows], dtype=torch.int32, device="cuda")
    lg = torch.empty((rows, L), device="cuda")
    pr = torch.empty((rows, L), dtype=torch.float64, device="cuda")
    sc = Scorer(bank, rows * L)
    for i in range(5):
        sc.score_list(slabs[i % 3], lg, pr, lst, cnt)
    torch.cuda.synchronize()
    best = 1e9
    for i in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        sc.score_list(slabs[i % 3], lg, pr, lst, cnt)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3)
    nbytes = rows * L * T * H * slabs[0].element_size()
    print(f"rows={rows} L={L} T={T} H={H} {dt}: {best:.1f} us  {nbytes / best / 1e3:.0f} GB/s", flush=True)
