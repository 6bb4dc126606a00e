"""Batched probe scoring on the GPU (K1) — the device side of the predictor seam.

``ProbeBank`` packs one linear probe per activation layer (the reference's
``MlpWeights`` with ``layer_dims=[]``, predictor.py:33-103) into the folded
form K1 consumes: ``wg = w * ln_gain`` (fp32, [L, H]) and
``c1 = w . ln_bias + b`` (computed in fp64, stored fp32), so
``logit = sum_h wg_h (m_h - mean(m)) / sqrt(var(m) + 1e-5) + c1`` — the same
algebra as predictor.py:134-148 with the token-window mean ``m`` in front.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib


@dataclass
class ProbeBank:
    wg: torch.Tensor      # [L, H] fp32 on device
    c1: torch.Tensor      # [L] fp32 on device
    H: int
    L: int

    @classmethod
    def from_linear(cls, w: np.ndarray, b, ln_gain=None, ln_bias=None,
                    device="cuda") -> "ProbeBank":
        """w: [L, H] (or [H]) probe weights, b: [L] biases; optional LN affine
        ([L, H] or [H]). Folding happens in fp64 on the host."""
        w = np.atleast_2d(np.asarray(w, dtype=np.float64))
        L, H = w.shape
        b = np.broadcast_to(np.asarray(b, dtype=np.float64).reshape(-1), (L,))
        g = np.ones((L, H)) if ln_gain is None else np.broadcast_to(
            np.asarray(ln_gain, dtype=np.float64), (L, H))
        beta = np.zeros((L, H)) if ln_bias is None else np.broadcast_to(
            np.asarray(ln_bias, dtype=np.float64), (L, H))
        wg = (w * g).astype(np.float32)
        c1 = (np.einsum("lh,lh->l", w, beta) + b).astype(np.float32)
        return cls(torch.from_numpy(np.ascontiguousarray(wg)).to(device),
                   torch.from_numpy(np.ascontiguousarray(c1)).to(device), H, L)

    @classmethod
    def from_mlp_weights(cls, probes, device="cuda") -> "ProbeBank":
        """One reference-style MlpWeights per layer, each a linear probe."""
        ws, bs, gs, betas = [], [], [], []
        for m in probes:
            if m.layer_dims or m.head_dim != 1:
                raise ValueError("ProbeBank holds linear probes (layer_dims=[], head_dim=1)")
            ws.append(np.asarray(m.weights[-1], dtype=np.float64).reshape(-1))
            bs.append(float(np.asarray(m.biases[-1]).reshape(-1)[0]))
            gs.append(np.ones(m.input_dim) if m.ln_gain is None else np.asarray(m.ln_gain))
            betas.append(np.zeros(m.input_dim) if m.ln_bias is None else np.asarray(m.ln_bias))
        return cls.from_linear(np.stack(ws), np.array(bs), np.stack(gs), np.stack(betas),
                               device=device)


class Scorer:
    """Owns the split-merge workspace for repeated K1 launches."""

    def __init__(self, bank: ProbeBank, max_units: int, nsplit: int = 0, threads: int = 0):
        _lib.require_cuda()
        self.lib = _lib.load()
        self.bank = bank
        self.nsplit = nsplit
        self.threads = threads
        dev = bank.wg.device
        nbytes = int(self.lib.duchess_score_workspace_bytes(max(max_units, 1), 16))
        self.workspace = torch.zeros(max(nbytes, 16), dtype=torch.uint8, device=dev)
        self.max_units = max_units

    def __call__(self, acts: torch.Tensor, out_logit: torch.Tensor, out_prob: torch.Tensor,
                 row_mask: torch.Tensor | None = None, stream=None) -> None:
        """acts: [rows, L, T, H] (any row stride, bf16 or fp32, CUDA).
        out_logit: [rows, L] fp32; out_prob: [rows, L] fp64."""
        _lib.require_cuda(acts)
        if acts.dim() != 4:
            raise ValueError("acts must be [rows, L, T, H]")
        rows, L, T, H = acts.shape
        if L != self.bank.L or H != self.bank.H:
            raise ValueError(f"activation shape (L={L}, H={H}) does not match probe bank "
                             f"(L={self.bank.L}, H={self.bank.H})")
        if rows * L > self.max_units:
            raise ValueError("more windows than the scorer workspace was sized for")
        if acts.stride(3) != 1:
            raise ValueError("hidden dimension must be contiguous")
        dtype = {torch.bfloat16: _lib.BF16, torch.float32: _lib.F32}.get(acts.dtype)
        if dtype is None:
            raise ValueError("activations must be bf16 or fp32")
        if row_mask is not None and (row_mask.dtype != torch.uint8 or row_mask.numel() < rows):
            raise ValueError("row_mask must be uint8 [rows]")
        st = acts.stride()
        _lib.check(self.lib.duchess_score(
            acts.data_ptr(), dtype, rows, L, T, H, st[0], st[1], st[2],
            self.bank.wg.data_ptr(), self.bank.c1.data_ptr(), _lib.ptr(row_mask),
            out_logit.data_ptr(), out_prob.data_ptr(), self.workspace.data_ptr(),
            self.workspace.numel(), self.nsplit, self.threads, _lib.stream_handle(stream)),
            "duchess_score")


    def score_list(self, acts: torch.Tensor, out_logit: torch.Tensor, out_prob: torch.Tensor,
                   row_list: torch.Tensor, row_count: torch.Tensor, stream=None) -> None:
        """Score only the rows in the device list row_list[:row_count[0]]
        (DuchessState.active_rows from duchess_advance); persistent TMA kernel."""
        _lib.require_cuda(acts)
        rows, L, T, H = acts.shape
        if L != self.bank.L or H != self.bank.H:
            raise ValueError(f"activation shape (L={L}, H={H}) does not match probe bank "
                             f"(L={self.bank.L}, H={self.bank.H})")
        dtype = {torch.bfloat16: _lib.BF16, torch.float32: _lib.F32}.get(acts.dtype)
        if dtype is None:
            raise ValueError("activations must be bf16 or fp32")
        if out_logit.dtype != torch.float32 or out_logit.numel() < rows * L:
            raise ValueError("out_logit must be fp32 with rows * L entries")
        if out_prob.dtype != torch.float64 or out_prob.numel() < rows * L:
            raise ValueError("out_prob must be fp64 with rows * L entries")
        st = acts.stride()
        _lib.check(self.lib.duchess_score_list(
            acts.data_ptr(), dtype, rows, L, T, H, st[0], st[1], st[2],
            self.bank.wg.data_ptr(), self.bank.c1.data_ptr(), row_list.data_ptr(),
            row_count.data_ptr(), out_logit.data_ptr(), out_prob.data_ptr(),
            _lib.stream_handle(stream)), "duchess_score_list")


    def score_active(self, acts: torch.Tensor, out_logit: torch.Tensor, out_prob: torch.Tensor,
                     engine, stream=None, no_input_wait: bool = False) -> None:
        """Score the survivors of the engine's round in flight (the active list
        duchess_advance / duchess_round left; parity chosen on the device).
        acts: [R*C, L, T, H] by branch slot. no_input_wait: the preceding
        kernel in the stream does not produce these inputs (the engine's K3
        launched with lead=True right after the round that did): stream at
        once, beside it (duchess_score_active_ex, DUCHESS_SCORE_NO_INPUT_WAIT)."""
        _lib.require_cuda(acts)
        rows, L, T, H = acts.shape
        if L != self.bank.L or H != self.bank.H:
            raise ValueError(f"activation shape (L={L}, H={H}) does not match probe bank "
                             f"(L={self.bank.L}, H={self.bank.H})")
        if rows != engine.R * engine.C:
            raise ValueError("acts must have R*C rows (one per branch slot)")
        if acts.stride(3) != 1:
            raise ValueError("hidden dimension must be contiguous")
        if out_logit.dtype != torch.float32 or out_logit.numel() < rows * L:
            raise ValueError("out_logit must be fp32 with rows * L entries")
        if out_prob.dtype != torch.float64 or out_prob.numel() < rows * L:
            raise ValueError("out_prob must be fp64 with rows * L entries")
        dtype = {torch.bfloat16: _lib.BF16, torch.float32: _lib.F32}.get(acts.dtype)
        if dtype is None:
            raise ValueError("activations must be bf16 or fp32")
        st = acts.stride()
        _lib.check(self.lib.duchess_score_active_ex(
            acts.data_ptr(), dtype, rows, L, T, H, st[0], st[1], st[2],
            self.bank.wg.data_ptr(), self.bank.c1.data_ptr(), engine.t["active_rows"].data_ptr(),
            engine.t["active_count"].data_ptr(), out_logit.data_ptr(), out_prob.data_ptr(),
            _lib.SCORE_NO_INPUT_WAIT if no_input_wait else 0, _lib.stream_handle(stream)),
            "duchess_score_active_ex")


def fill_windows(acts: torch.Tensor, seed: int, row_req=None, row_tmpl=None, row_pos=None,
                 row_mask=None, stream=None) -> None:
    """Write counter-hashed synthetic activations (oracle/activations.py
    regenerates them bit for bit) into acts [rows, L, T, H]."""
    _lib.require_cuda(acts)
    lib = _lib.load()
    rows, L, T, H = acts.shape
    dtype = {torch.bfloat16: _lib.BF16, torch.float32: _lib.F32}[acts.dtype]
    st = acts.stride()
    _lib.check(lib.duchess_fill_activations(
        acts.data_ptr(), dtype, rows, L, T, H, st[0], st[1], st[2], seed & ((1 << 64) - 1),
        _lib.ptr(row_req), _lib.ptr(row_tmpl), _lib.ptr(row_pos), _lib.ptr(row_mask),
        _lib.stream_handle(stream)), "duchess_fill_activations")
