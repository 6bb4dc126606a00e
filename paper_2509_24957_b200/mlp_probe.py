"""Tensor-core MLP probe (``duchess_mlp_probe_tc``): the paper's MLP probe
 batched over many activation vectors as a tcgen05 GEMM with the
LayerNorm, bias, ReLU and 1-dim head fused into the epilogue.

Parameters come from a reference-style ``MlpWeights`` with one hidden layer
(ReLU), optional input LayerNorm and optional inference batch-norm (folded into
the hidden affine map on the host). W1 * ln_gain is stored bf16 (the tensor-core
operand type); the fold constants are computed from those bf16 values so the
only deviation from fp64 on the same bf16 operands is fp32 accumulation.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _lib
from .hostmath import bf16_round_np

BN_TILE, BK = 256, 64


class TensorCoreMlpProbe:
    def __init__(self, weights, device="cuda"):
        _lib.require_cuda()
        self.lib = _lib.load()
        if len(weights.layer_dims) != 1 or weights.head_dim != 1:
            raise ValueError("tensor-core probe supports one hidden layer and a 1-dim head")
        if weights.activations[0] != "relu":
            raise ValueError("tensor-core probe supports a ReLU hidden layer")
        K, NH = weights.input_dim, weights.layer_dims[0]
        if K % BK:
            raise ValueError(f"input_dim must be a multiple of {BK}")
        W1 = np.asarray(weights.weights[0], dtype=np.float64)
        b1 = np.asarray(weights.biases[0], dtype=np.float64)
        if weights.bn_mean is not None:               # inference BN is affine: fold it
            scale = np.asarray(weights.bn_gain[0]) / np.sqrt(np.asarray(weights.bn_var[0]) + 1e-5)
            W1 = W1 * scale[:, None]
            b1 = (b1 - np.asarray(weights.bn_mean[0])) * scale + np.asarray(weights.bn_bias[0])
        g = np.ones(K) if weights.ln_gain is None else np.asarray(weights.ln_gain, dtype=np.float64)
        beta = np.zeros(K) if weights.ln_bias is None else np.asarray(weights.ln_bias, dtype=np.float64)
        NHp = -(-NH // BN_TILE) * BN_TILE
        W1g = np.zeros((NHp, K))
        W1g[:NH] = bf16_round_np(W1 * g[None, :])
        c = np.zeros(NHp)
        c[:NH] = W1 @ beta + b1
        w2 = np.zeros(NHp)
        w2[:NH] = np.asarray(weights.weights[1], dtype=np.float64).reshape(-1)
        self.K, self.NH, self.NHp = K, NH, NHp
        self.W1g = W1g                                  # bf16-exact values (fp64 array)
        self.c, self.w2 = c, w2
        self.b2 = float(np.asarray(weights.biases[1]).reshape(-1)[0])
        self.s = W1g.sum(axis=1)
        dev = torch.device(device)
        self.d_w1 = torch.from_numpy(W1g.astype(np.float32)).to(dev).to(torch.bfloat16).contiguous()
        self.d_s = torch.from_numpy(self.s.astype(np.float32)).to(dev)
        self.d_c = torch.from_numpy(c.astype(np.float32)).to(dev)
        self.d_w2 = torch.from_numpy(w2.astype(np.float32)).to(dev)
        self._ws = None                                 # zeroed workspace, grown on demand

    def __call__(self, X: torch.Tensor, out_logit: torch.Tensor | None = None,
                 out_prob: torch.Tensor | None = None, stream=None):
        """X: [M, K] bf16 contiguous (CUDA) -> (logits fp32 [M], probs fp64 [M])."""
        if X.dtype != torch.bfloat16 or X.dim() != 2 or X.shape[1] != self.K or not X.is_contiguous():
            raise ValueError(f"X must be a contiguous bf16 [M, {self.K}] tensor")
        M = X.shape[0]
        if out_logit is None:
            out_logit = torch.empty(M, dtype=torch.float32, device=X.device)
        if out_prob is None:
            out_prob = torch.empty(M, dtype=torch.float64, device=X.device)
        need = int(self.lib.duchess_mlp_probe_tc_workspace_bytes(M, self.NHp))
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.zeros(need, dtype=torch.uint8, device=X.device)
        _lib.check(self.lib.duchess_mlp_probe_tc(
            X.data_ptr(), M, self.K, self.d_w1.data_ptr(), self.NHp, self.d_s.data_ptr(),
            self.d_c.data_ptr(), self.d_w2.data_ptr(), self.b2, out_logit.data_ptr(),
            out_prob.data_ptr(), self._ws.data_ptr(), self._ws.numel(),
            _lib.stream_handle(stream)), "duchess_mlp_probe_tc")
        return out_logit, out_prob

    def flops(self, M: int) -> float:
        return 2.0 * M * self.K * self.NHp
