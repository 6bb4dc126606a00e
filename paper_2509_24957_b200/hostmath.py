"""Small numeric helpers shared by host-side packing code (not the oracle)."""

from __future__ import annotations

import numpy as np


def bf16_round_np(x) -> np.ndarray:
    """Round to the nearest bf16 (ties to even), returned as float64 values."""
    f = np.ascontiguousarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    return (u.astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)
