"""Batched difficulty classifier on the tensor cores.

The reference predicts a request's difficulty with ``predict_difficulty("mlp")``:
the complexity MLP (PAPER.md:464 — 4096 -> 2048 -> 1024 -> 512 -> 5, batch-norm
and GeLU, softmax head) run through ``mlp_forward`` (predictor.py:126-151) one
vector at a time in fp64, level = argmax + 1 (predictor.py:398-402). Batched
over many requests the hidden layers are real GEMMs, so they run as tcgen05
layers (``duchess_tc_linear``: bf16 operands, fp32 accumulation, LayerNorm /
bias / batch-norm / GeLU fused in the TMEM epilogue) and the 5-way head as
``duchess_head_logits``.

The input LayerNorm runs as its own pass (``duchess_row_normalize``: fp64
statistics, z = (x - mean) / std written bf16), so the first tensor-core layer
sees zero-mean unit-scale rows whatever the raw activations' offset (folding
mean * S into the epilogue cancels badly in fp32 for rows with a large common
offset). The LN affine (gain, bias) is folded into that layer's weights / bias.

Levels are discrete, so bf16 rounding must never flip an argmax: a row whose
top-two logits are closer than ``margin`` is recomputed by the fp64 device
forward (``duchess_mlp_forward``, the facade's ``mlp_forward``). Because every
row reaches the tensor cores LayerNorm-normalised, the logit error does not
scale with the raw input; the default margin is derived per classifier at
construction: 8x the largest |tensor-core - fp64| logit gap over a calibration
batch of 512 N(0, 1) rows with 1% outlier channels at 20x (at least 0.05), so
a flip would need an error 4x beyond anything measured on either side of a tie.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .predictor import ACTIVATION_KINDS, BATCHNORM_EPS, MlpWeights, WeightFormatError, mlp_forward_batch


def _bf16(a: np.ndarray, device) -> torch.Tensor:
    return torch.tensor(np.asarray(a, dtype=np.float32), device=device).to(torch.bfloat16).contiguous()


def _f32(a, device) -> torch.Tensor:
    return torch.tensor(np.asarray(a, dtype=np.float64).astype(np.float32), device=device)


class TensorCoreClassifier:
    """mlp_forward for a classifier head (head_dim > 1) batched over rows on
    tcgen05. Needs input_dim % 64 == 0 and hidden widths % 256 == 0."""

    def __init__(self, weights: MlpWeights, device="cuda", margin: float | None = None):
        _lib.require_cuda()
        weights.validate()
        if weights.head_dim < 2:
            raise ValueError("TensorCoreClassifier is for softmax heads (head_dim > 1)")
        if not weights.layer_dims:
            raise ValueError("the tensor-core path needs at least one hidden layer")
        if weights.input_dim % 64 or any(d % 256 for d in weights.layer_dims):
            raise ValueError("input_dim must be a multiple of 64 and hidden widths of 256")
        self.lib = _lib.load()
        self.weights = weights
        self.device = torch.device(device)
        dev = self.device
        d0 = weights.input_dim
        g = np.ones(d0) if weights.ln_gain is None else np.asarray(weights.ln_gain, np.float64)
        bl = np.zeros(d0) if weights.ln_bias is None else np.asarray(weights.ln_bias, np.float64)
        self.layers = []
        for k, width in enumerate(weights.layer_dims):
            W = np.asarray(weights.weights[k], dtype=np.float64)
            b = np.asarray(weights.biases[k], dtype=np.float64)
            if k == 0:          # LN affine folded into the first layer (input normalised)
                Wd, S, C = _bf16(W * g[None, :], dev), None, _f32(W @ bl + b, dev)
            else:
                Wd, S, C = _bf16(W, dev), None, _f32(b, dev)
            if weights.has_batchnorm:
                bs = np.asarray(weights.bn_gain[k], np.float64) / np.sqrt(
                    np.asarray(weights.bn_var[k], np.float64) + BATCHNORM_EPS)
                bt = np.asarray(weights.bn_bias[k], np.float64) - np.asarray(
                    weights.bn_mean[k], np.float64) * bs
            else:
                bs, bt = np.ones(width), np.zeros(width)
            act = ACTIVATION_KINDS.index(weights.activations[k]) + 1    # 1 relu, 2 gelu
            self.layers.append((Wd, S, C, _f32(bs, dev), _f32(bt, dev), act, width))
        self.head_w = _f32(weights.weights[-1], dev).contiguous()
        self.head_b = _f32(weights.biases[-1], dev)
        self.margin = self.calibrate_margin() if margin is None else float(margin)

    def calibrate_margin(self, n: int = 512, seed: int = 0) -> float:
        """8x the largest tensor-core vs fp64 logit gap on normalised-scale
        calibration rows (at least 0.05); see the module docstring."""
        rng = np.random.default_rng(seed)
        X = rng.standard_normal((n, self.weights.input_dim))
        X[:, rng.random(self.weights.input_dim) < 0.01] *= 20.0
        tc = self.logits(X).double().cpu().numpy()
        ref, _ = mlp_forward_batch(self.weights, X)
        self.calibration_error = float(np.abs(tc - ref).max())
        return max(8.0 * self.calibration_error, 0.05)

    def logits(self, X) -> torch.Tensor:
        """X [M, input_dim] (numpy or torch) -> fp32 logits [M, head_dim] on the device."""
        x = torch.as_tensor(X, device=self.device)
        if x.dim() != 2 or x.shape[1] != self.weights.input_dim:
            raise WeightFormatError(f"activation shape {tuple(x.shape[1:])} does not match "
                                    f"expected ({self.weights.input_dim},)")
        # fp64 inputs stay fp64 until normalised (a large common offset would
        # swallow an fp32 row's signal); bf16 / fp32 rows are read as they are;
        # anything else is read as fp32
        K = x.shape[1]
        if x.dtype == torch.bfloat16 and K % 8 == 0 and K <= 8192:
            xf, dt = x.contiguous(), _lib.BF16
        elif x.dtype == torch.float64:
            xf, dt = x.contiguous(), _lib.F64
        else:
            xf, dt = x.to(torch.float32).contiguous(), _lib.F32
        M = xf.shape[0]
        stream = _lib.stream_handle()
        h = torch.empty((M, K), dtype=torch.bfloat16, device=self.device)
        _lib.check(self.lib.duchess_row_normalize(xf.data_ptr(), dt, M, K, h.data_ptr(), stream),
                   "duchess_row_normalize")
        for Wd, _S, C, BS, BT, act, width in self.layers:
            out = torch.empty((M, width), dtype=torch.bfloat16, device=self.device)
            _lib.check(self.lib.duchess_tc_linear(
                h.data_ptr(), M, h.shape[1], Wd.data_ptr(), width, 0, None, C.data_ptr(),
                BS.data_ptr(), BT.data_ptr(), act, out.data_ptr(), None, 0, stream),
                "duchess_tc_linear")
            h = out
        logits = torch.empty((M, self.weights.head_dim), dtype=torch.float32, device=self.device)
        _lib.check(self.lib.duchess_head_logits(
            h.data_ptr(), M, h.shape[1], self.head_w.data_ptr(), self.head_b.data_ptr(),
            self.weights.head_dim, logits.data_ptr(), stream), "duchess_head_logits")
        return logits

    def predict_levels(self, X) -> np.ndarray:
        """predict_difficulty("mlp") for every row: argmax + 1 (predictor.py:398-402),
        near ties (top-two logits within margin) recomputed in fp64 on the device."""
        X = np.asarray(X, dtype=np.float64)
        lg = self.logits(X).cpu().numpy()
        top2 = np.sort(lg, axis=1)[:, -2:]
        levels = lg.argmax(axis=1) + 1
        close = np.nonzero(top2[:, 1] - top2[:, 0] < self.margin)[0]
        if len(close):
            _, probs = mlp_forward_batch(self.weights, X[close])
            levels[close] = probs.argmax(axis=1) + 1
        self.last_fallback = len(close)
        return levels
