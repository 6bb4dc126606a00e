"""One K1 launch over a fully active C2 slab (4096 windows x 32 x 4096 bf16 =
1 GiB algorithmic bytes) for ncu capture; prints the launch's algorithmic bytes."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2509_24957_b200.probe import ProbeBank, Scorer, fill_windows  # noqa: E402

rows, T, H = 4096, 32, 4096
rng = np.random.default_rng(0)
bank = ProbeBank.from_linear(rng.normal(0, 1.5 / 64, (1, H)), [0.0])
slab = torch.empty((rows, 1, T, H), dtype=torch.bfloat16, device="cuda")
fill_windows(slab, 1)
lst = torch.arange(rows, dtype=torch.int32, device="cuda")
cnt = torch.tensor([rows], dtype=torch.int32, device="cuda")
logit = torch.empty((rows, 1), device="cuda")
prob = torch.empty((rows, 1), dtype=torch.float64, device="cuda")
sc = Scorer(bank, rows)
for _ in range(3):
    sc.score_list(slab, logit, prob, lst, cnt)
torch.cuda.synchronize()
print("algorithmic_bytes", rows * T * H * 2)
