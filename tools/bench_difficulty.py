"""Throughput of the tensor-core difficulty classifier (complexity MLP
4096 -> 2048 -> 1024 -> 512 -> 5, BN + GeLU) vs the fp64 per-row device forward."""
import sys
import time
import numpy as np
import torch
sys.path.insert(0, ".")
from tests.test_gpu_difficulty import activations, complexity_mlp  # noqa: E402
from paper_2509_24957_b200.difficulty import TensorCoreClassifier  # noqa: E402
from paper_2509_24957_b200.predictor import mlp_forward_batch  # noqa: E402

dims = (4096, 2048, 1024, 512)
w = complexity_mlp(1, dims)
clf = TensorCoreClassifier(w)
flops_row = 2 * (4096 * 2048 + 2048 * 1024 + 1024 * 512)
for M in (4096, 32768):
    X = torch.tensor(activations(2, M, 4096), dtype=torch.float32, device="cuda").to(torch.bfloat16)
    for _ in range(3):
        clf.logits(X)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    e0.record()
    for _ in range(n):
        clf.logits(X)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"tc M={M}: {ms:.3f} ms, {M / ms * 1e3 / 1e6:.2f} M requests/s, "
          f"{flops_row * M / ms / 1e9:.0f} TFLOP/s")
Xs = activations(3, 256, 4096)
t0 = time.perf_counter()
mlp_forward_batch(w, Xs)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"fp64 per-row device forward: {256 / dt:.0f} requests/s")
