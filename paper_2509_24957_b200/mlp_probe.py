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


def _bn_fold(w: np.ndarray, b: np.ndarray, weights, k: int):
    """Inference batch-norm of hidden layer k folded into its affine map
    (predictor.py:141-143: (h - mean) / sqrt(var + eps) * gain + bias)."""
    if weights.bn_mean is None:
        return w, b
    scale = np.asarray(weights.bn_gain[k]) / np.sqrt(np.asarray(weights.bn_var[k]) + 1e-5)
    return w * scale[:, None], (b - np.asarray(weights.bn_mean[k])) * scale + \
        np.asarray(weights.bn_bias[k])


class MlpProbeBank:
    """The paper's correctness probe — input LayerNorm -> Linear -> ReLU ->
    Linear -> ReLU -> 1 (5120 -> 2048 -> 1024 -> 1 at the
    C3 shape), evaluated by the reference one vector at a time in fp64
    (predictor.py:126-151) — for L probe layers at once on the tensor cores,
    two launches for all layers:

      1. ``duchess_tc_linear_grouped``: h1 = relu(LN(x_l) W1_l^T + b1_l) for
         every layer l, reading x straight from the engine's activation slab
         [rows, L, H] (3D TMA map, one token per layer), LN folded into the
         epilogue, h1 stored bf16 [L, rows, 2048];
      2. ``duchess_mlp_probe_tc_grouped`` (ln = 0): h2 = relu(h1 W2_l^T + b2_l)
         with the 1-dim head w3_l . h2 + b3_l fused into the epilogue (h2
         never reaches HBM), logits fp32 / probabilities fp64 [rows, L].

    Operands are bf16 (X as read, W1 * ln_gain, h1, W2), accumulation fp32.
    A one-hidden-layer MLP runs as launch 2 alone with the LN folded (ln = 1).
    """

    def __init__(self, probes, device="cuda"):
        _lib.require_cuda()
        self.lib = _lib.load()
        probes = list(probes)
        if not probes:
            raise ValueError("at least one probe")
        dims = {(p.input_dim, tuple(p.layer_dims), p.head_dim, tuple(p.activations))
                for p in probes}
        if len(dims) != 1:
            raise ValueError("all probe layers must share one architecture")
        K, hidden, head, acts = dims.pop()
        if head != 1 or len(hidden) not in (1, 2) or any(a != "relu" for a in acts):
            raise ValueError("MlpProbeBank runs ReLU MLPs with one or two hidden layers and a "
                             "1-dim head")
        if K % BK or any(h % BN_TILE for h in hidden) or (len(hidden) == 2 and hidden[0] % BK):
            raise ValueError(f"input_dim must be a multiple of {BK}, hidden widths of {BN_TILE}")
        self.G, self.K, self.hidden = len(probes), K, list(hidden)
        dev = torch.device(device)
        self.device = dev
        W1s, S1, C1, Wn, cn, wh, bh = [], [], [], [], [], [], []
        for p in probes:
            g = np.ones(K) if p.ln_gain is None else np.asarray(p.ln_gain, dtype=np.float64)
            beta = np.zeros(K) if p.ln_bias is None else np.asarray(p.ln_bias, dtype=np.float64)
            w1, b1 = _bn_fold(np.asarray(p.weights[0], dtype=np.float64),
                              np.asarray(p.biases[0], dtype=np.float64), p, 0)
            w1g = bf16_round_np(w1 * g[None, :])
            W1s.append(w1g)
            S1.append(w1g.sum(axis=1))
            C1.append(w1 @ beta + b1)
            if len(hidden) == 2:
                w2, b2 = _bn_fold(np.asarray(p.weights[1], dtype=np.float64),
                                  np.asarray(p.biases[1], dtype=np.float64), p, 1)
                Wn.append(bf16_round_np(w2))
                cn.append(b2)
            wh.append(np.asarray(p.weights[-1], dtype=np.float64).reshape(-1))
            bh.append(float(np.asarray(p.biases[-1]).reshape(-1)[0]))
        f32 = lambda a: torch.from_numpy(np.ascontiguousarray(np.concatenate(a)).astype(np.float32)).to(dev)
        bf = lambda a: torch.from_numpy(np.ascontiguousarray(np.concatenate(a)).astype(np.float32)).to(dev).to(torch.bfloat16)
        self.host = dict(W1=W1s, S1=S1, C1=C1, W2=Wn, c2=cn, w3=wh, b3=bh)
        self.d_w1, self.d_s1, self.d_c1 = bf(W1s), f32(S1), f32(C1)
        self.d_head = f32(wh)
        self.d_bh = torch.tensor(bh, dtype=torch.float32, device=dev)
        if len(hidden) == 2:
            self.d_w2, self.d_c2 = bf(Wn), f32(cn)
            self.d_ones = torch.ones(self.G * hidden[0], dtype=torch.float32, device=dev)
            self.d_zeros = torch.zeros(self.G * hidden[0], dtype=torch.float32, device=dev)
        self._h1 = None
        self._ws1 = self._ws2 = None
        self.L, self.H = self.G, self.K          # the ProbeBank shape the engine expects

    @classmethod
    def paper_probes(cls, L: int, H: int, seed: int = 0, hidden=(2048, 1024)):
        """L random-init probes of the paper's architecture:
        LN affine, He-scaled ReLU layers, a small head (reference-style
        MlpWeights; there are no trained checkpoints offline)."""
        from .predictor import MlpWeights
        rng = np.random.default_rng(seed)
        out = []
        for _ in range(L):
            dims = [H, *hidden, 1]
            ws = [rng.normal(0.0, np.sqrt(2.0 / dims[k]), (dims[k + 1], dims[k]))
                  for k in range(len(dims) - 1)]
            ws[-1] *= 0.5
            bs = [rng.normal(0.0, 0.05, dims[k + 1]) for k in range(len(dims) - 1)]
            out.append(MlpWeights(H, list(hidden), 1, ["relu"] * len(hidden), ws, bs,
                                  rng.uniform(0.5, 1.5, H), rng.uniform(-0.1, 0.1, H)))
        return out

    def _grow(self, name, nbytes):
        buf = getattr(self, name)
        if buf is None or buf.numel() < nbytes:
            buf = torch.zeros(max(nbytes, 16), dtype=torch.uint8, device=self.device)
            setattr(self, name, buf)
        return buf

    def __call__(self, X: torch.Tensor, out_logit: torch.Tensor, out_prob: torch.Tensor,
                 stream=None):
        """X: bf16 [M, G, K] contiguous (the activation slab [rows, L, 1, H]
        viewed per layer) -> out_logit fp32 / out_prob fp64, [M, G] each."""
        G, K = self.G, self.K
        if X.dtype != torch.bfloat16 or not X.is_contiguous() or X.numel() % (G * K):
            raise ValueError(f"X must be a contiguous bf16 [M, {G}, {K}] tensor")
        M = X.numel() // (G * K)
        if out_logit.numel() < M * G or out_prob.numel() < M * G:
            raise ValueError("outputs must hold [M, G] entries")
        st = _lib.stream_handle(stream)
        if len(self.hidden) == 1:
            NH = self.hidden[0]
            ws = self._grow("_ws2", int(self.lib.duchess_mlp_probe_tc_grouped_workspace_bytes(M, G, NH)))
            _lib.check(self.lib.duchess_mlp_probe_tc_grouped(
                X.data_ptr(), M, K, G, 1, 1, self.d_w1.data_ptr(), NH, self.d_s1.data_ptr(),
                self.d_c1.data_ptr(), self.d_head.data_ptr(), self.d_bh.data_ptr(),
                out_logit.data_ptr(), out_prob.data_ptr(), ws.data_ptr(), ws.numel(), st),
                "duchess_mlp_probe_tc_grouped")
            return out_logit, out_prob
        N1, N2 = self.hidden
        if self._h1 is None or self._h1.numel() < G * M * N1:
            self._h1 = torch.empty(G * M * N1, dtype=torch.bfloat16, device=self.device)
        ws1 = self._grow("_ws1", int(self.lib.duchess_tc_linear_grouped_workspace_bytes(M, G, N1)))
        _lib.check(self.lib.duchess_tc_linear_grouped(
            X.data_ptr(), M, K, G, 1, self.d_w1.data_ptr(), N1, 1, self.d_s1.data_ptr(),
            self.d_c1.data_ptr(), self.d_ones.data_ptr(), self.d_zeros.data_ptr(), 1,
            self._h1.data_ptr(), ws1.data_ptr(), ws1.numel(), st), "duchess_tc_linear_grouped")
        ws2 = self._grow("_ws2", int(self.lib.duchess_mlp_probe_tc_grouped_workspace_bytes(M, G, N2)))
        _lib.check(self.lib.duchess_mlp_probe_tc_grouped(
            self._h1.data_ptr(), M, N1, G, 0, 0, self.d_w2.data_ptr(), N2, None,
            self.d_c2.data_ptr(), self.d_head.data_ptr(), self.d_bh.data_ptr(),
            out_logit.data_ptr(), out_prob.data_ptr(), ws2.data_ptr(), ws2.numel(), st),
            "duchess_mlp_probe_tc_grouped")
        return out_logit, out_prob

    def flops(self, M: int) -> float:
        dims = [self.K, *self.hidden]
        return 2.0 * M * self.G * (sum(dims[k] * dims[k + 1] for k in range(len(dims) - 1))
                                   + dims[-1])


class MlpScorer:
    """Engine-facing scorer for an MlpProbeBank (the serving loop's K1 slot):
    every branch slot's last-token window [R*C, L, 1, H] bf16 through the
    paper's probe for all L layers (dense over the slots: GEMM tiles need
    contiguous rows; inactive slots' scores are computed and ignored, the
    decision kernel reads survivors only)."""

    def __init__(self, bank: MlpProbeBank):
        self.bank = bank

    def score_active(self, acts: torch.Tensor, out_logit: torch.Tensor, out_prob: torch.Tensor,
                     engine, stream=None) -> None:
        rows, L, T, H = acts.shape
        if L != self.bank.G or H != self.bank.K or T != 1:
            raise ValueError(f"activations must be [rows, {self.bank.G}, 1, {self.bank.K}] "
                             f"(the last token, PAPER.md:150)")
        if rows != engine.R * engine.C:
            raise ValueError("acts must have R*C rows (one per branch slot)")
        self.bank(acts.view(rows, L, H), out_logit, out_prob, stream)
