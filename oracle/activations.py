"""Bit-exact CPU regeneration of the synthetic activation windows.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). Mirrors
paper_2509_24957_b200/csrc/common.cuh (mix64 / row_key / synth_value /
f32_to_bf16_rne): windows are keyed by (seed, request, template index,
position, layer), which is unique per branch-step because branch_id ==
template_index (reference orchestrator.py:260-266) and every survivor advances
at least one token per round (orchestrator.py:273-279).
"""

from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1
ACT_SCALE = np.frombuffer(np.uint32(0x37DDB3D7).tobytes(), dtype=np.float32)[0]
OUTLIER_GAIN = np.float32(20.0)


def mix64_int(z: int) -> int:
    z = (z + 0x9E3779B97F4A7C15) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def row_key(seed: int, req: int, tmpl: int, pos: int, layer: int) -> int:
    k = mix64_int(seed & MASK64)
    k = mix64_int(k ^ (req & MASK64))
    k = mix64_int(k ^ (tmpl & 0xFFFFFFFF))
    return mix64_int(k ^ (((pos & 0xFFFFFFFF) << 8) | layer))


def _mix64_np(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def bf16_round(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 round-to-nearest-even, returned as fp32 values."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    return (u.astype(np.uint32) << np.uint32(16)).view(np.float32)


def synth_window(seed: int, req: int, tmpl: int, pos: int, layer: int, T: int, H: int,
                 bf16: bool) -> np.ndarray:
    """[T, H] float32 window exactly as the GPU fill kernel stores it."""
    rk = np.uint64(row_key(seed, req, tmpl, pos, layer))
    t = np.arange(T, dtype=np.uint64)[:, None]
    h = np.arange(H, dtype=np.uint64)[None, :]
    e = _mix64_np(rk ^ ((t << np.uint64(32)) | h))
    m = np.uint64(0xFFFF)
    s = ((e & m).astype(np.int64) + ((e >> np.uint64(16)) & m).astype(np.int64)
         + ((e >> np.uint64(32)) & m).astype(np.int64) + (e >> np.uint64(48)).astype(np.int64))
    x = (s - 131070).astype(np.float32) * ACT_SCALE
    out = (np.arange(H) & 511) == 257
    x[:, out] = x[:, out] * OUTLIER_GAIN
    return bf16_round(x) if bf16 else x
