"""Probe training (K4): logistic regression of branch correctness on pooled
activations, data-parallel over GPUs.

Absent from the reference; the paper trains its probes with BCE
(PAPER.md:169, :448-450). One step = the fused gradient kernel over this
rank's row shard (``duchess_lr_grad``: one HBM pass, TMA-bulk staged), an
all-reduce of the H+1 gradient over NCCL (the only collective on the path;
32 KB at H=8192, latency-bound), and an SGD update on device.
"""

from __future__ import annotations

import torch

from . import _lib


class LogisticProbeTrainer:
    def __init__(self, H: int, device="cuda", group=None, lr: float = 0.1):
        _lib.require_cuda()
        self.lib = _lib.load()
        self.H = H
        self.device = torch.device(device)
        self.group = group
        self.lr = lr
        self.w = torch.zeros(H + 1, dtype=torch.float32, device=self.device)
        self.grad = torch.zeros(H + 1, dtype=torch.float32, device=self.device)
        ws = int(self.lib.duchess_lr_grad_workspace_bytes(H))
        self.ws = torch.zeros(max(ws, 16), dtype=torch.uint8, device=self.device)

    def local_grad(self, X: torch.Tensor, y: torch.Tensor, inv_n: float, stream=None) -> torch.Tensor:
        """grad = inv_n * [X^T (sigmoid(Xw+b) - y), sum(...)] over this shard."""
        if X.dim() != 2 or X.shape[1] != self.H or not X.is_contiguous():
            raise ValueError(f"X must be a contiguous [N, {self.H}] tensor")
        dtype = {torch.bfloat16: _lib.BF16, torch.float32: _lib.F32}.get(X.dtype)
        if dtype is None:
            raise ValueError("X must be bf16 or fp32")
        _lib.check(self.lib.duchess_lr_grad(
            X.data_ptr(), dtype, y.data_ptr(), self.w.data_ptr(), X.shape[0], self.H,
            float(inv_n), self.grad.data_ptr(), self.ws.data_ptr(), self.ws.numel(),
            _lib.stream_handle(stream)), "duchess_lr_grad")
        return self.grad

    def step(self, X: torch.Tensor, y: torch.Tensor, n_total: int, stream=None) -> torch.Tensor:
        """One full-batch step over the global N = n_total rows (this rank holds X)."""
        g = self.local_grad(X, y, 1.0 / n_total, stream)
        allreduce_sum(g, self.group)
        _lib.check(self.lib.duchess_sgd_update(self.w.data_ptr(), g.data_ptr(), self.H + 1,
                                               float(self.lr), _lib.stream_handle(stream)),
                   "duchess_sgd_update")
        return g


from .distributed import allreduce_sum, shard_range as shard_rows  # noqa: E402,F401
