"""CPU restatements of the north-star extensions that have no reference code.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). The reference forks by
accounting only (orchestrator.py:254-268, :384: the child resumes at
``source.position`` without re-charging the prefix; PAPER.md:466 relies on vLLM
prefix caching) and ships no training. These serial restatements
define the semantics the CUDA kernels must match bit for bit (K3) or within
fp32 reduction tolerance (K4).
"""

from __future__ import annotations

import numpy as np


def cow_fork_ref(forks, counts, block_table, refcount, free_list, cursor, kv_pool,
                 kv_bytes_per_token: int, block_tokens: int, rows_per_group: int):
    """Serial copy-on-write block-table fork, in (group, record) order.

    forks: int array [n_groups, group_cap, 4] of (child, source, table_root,
    prefix_tokens); counts[g] valid records per group (None = all).
    block_table: [rows, stride] int32 (row = g * rows_per_group + branch id).
    For each fork: the child row gets the root's first prefix // block_tokens
    entries (refcount += 1 each); a partial tail takes free_list[cursor + k]
    (k = rank among tail-needing forks), gets refcount 1 and a copy of the
    root's first prefix % block_tokens tokens of KV bytes; the rest of the
    child row is -1. Returns (table, refcount, cursor, kv_pool, status)."""
    table = block_table.copy()
    ref = refcount.copy()
    kv = None if kv_pool is None else kv_pool.copy()
    n_groups, group_cap = forks.shape[0], forks.shape[1]
    block_bytes = kv_bytes_per_token * block_tokens
    status = 0
    for g in range(n_groups):
        n = group_cap if counts is None else int(min(max(counts[g], 0), group_cap))
        for k in range(n):
            child, _src, root, prefix = (int(v) for v in forks[g, k])
            base = g * rows_per_group
            src_row = table[base + root].copy()
            n_full, tail = divmod(prefix, block_tokens)
            new = np.full(table.shape[1], -1, dtype=table.dtype)
            new[:n_full] = src_row[:n_full]
            for blk in src_row[:n_full]:
                ref[blk] += 1
            if tail:
                if cursor < len(free_list):
                    blk = int(free_list[cursor])
                    cursor += 1
                    new[n_full] = blk
                    ref[blk] = 1
                    if kv is not None:
                        s = int(src_row[n_full]) * block_bytes
                        d = blk * block_bytes
                        nb = tail * kv_bytes_per_token
                        kv[d:d + nb] = kv[s:s + nb]
                else:
                    status = 1
            table[base + child] = new
    return table, ref, cursor, kv, status


def lr_grad_ref(X: np.ndarray, y: np.ndarray, w: np.ndarray) -> np.ndarray:
    """Logistic-regression gradient of the mean BCE, fp64: w is [H+1] (bias
    last); returns [H+1] = (X^T r / N, sum(r) / N) with r = sigmoid(Xw+b) - y."""
    Xd = np.asarray(X, dtype=np.float64)
    z = Xd @ np.asarray(w[:-1], dtype=np.float64) + float(w[-1])
    r = 1.0 / (1.0 + np.exp(-z)) - np.asarray(y, dtype=np.float64)
    n = Xd.shape[0]
    return np.concatenate([Xd.T @ r, [r.sum()]]) / n


def difficulty_order_ref(levels, arrivals) -> list[int]:
    """Python sorted() by (level, arrival, order): the sequence of repeated
    scheduler.py:60-96 next_request pops over one snapshot (keys are unique)."""
    return sorted(range(len(levels)), key=lambda j: (levels[j], arrivals[j], j))
