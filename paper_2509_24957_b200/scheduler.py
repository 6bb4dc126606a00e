"""Inter-request scheduling (mirrors reference scheduler.py).

Difficulty ordering is the device segmented sort ``duchess_sort_difficulty``
over 64-bit keys ``level << 61 | arrival << 21 | order``. The keys are unique,
so sorting one queue snapshot gives exactly the sequence of repeated
``next_request`` pops (scheduler.py:60-96); ``next_request`` itself is that
sort over the eligible entries, popping the first.
"""

from __future__ import annotations

import random
from dataclasses import dataclass

import numpy as np

from .workload import RequestTrace

FCFS = "fcfs"
EASIEST_ACTUAL = "easiest-actual"
EASIEST_PREDICTED = "easiest-predicted"
SCHEDULES = (FCFS, EASIEST_ACTUAL, EASIEST_PREDICTED)

SEGMENT_MAX = 4096          # keys per device segment (one CTA, shared memory)
_ARRIVAL_BITS, _ORDER_BITS = 40, 21


@dataclass(frozen=True)
class ArrivalConfig:
    rate_qpm: float
    n_requests: int
    seed: int = 0

    def __post_init__(self) -> None:
        if self.rate_qpm <= 0:
            raise ValueError("rate_qpm must be > 0")
        if self.n_requests < 1:
            raise ValueError("n_requests must be >= 1")


def gen_arrivals(config: ArrivalConfig) -> list:
    """Strictly increasing Poisson arrival times in ms (scheduler.py:35-48)."""
    rng = random.Random(config.seed)
    gap = 60000.0 / config.rate_qpm
    out, t, prev = [], 0.0, -1
    for _ in range(config.n_requests):
        t += rng.expovariate(1.0 / gap)
        prev = max(int(round(t)), prev + 1)
        out.append(prev)
    return out


@dataclass
class QueueEntry:
    trace: RequestTrace
    arrival: int
    order: int
    prefill_done: int | None = None
    predicted_difficulty: int | None = None


def pack_keys(levels, arrivals, orders, tiebreak=None) -> np.ndarray:
    """64-bit sort keys ordering like the tuples (level, arrival, order)
    (scheduler.py:84-90). Fast path: level < 8, arrival < 2^40 ms,
    order < 2^21 packed directly; otherwise each field is replaced by its
    dense rank (order-preserving) and packed with just enough bits, so any
    integer fields sort exactly as the reference's tuples. `tiebreak` (e.g.
    the queue index) appends a last field so equal tuples keep the order the
    reference's strict `<` scan gives them (the first in the queue wins)."""
    cols = [levels, arrivals, orders] + ([] if tiebreak is None else [tiebreak])
    cols = [np.asarray([int(x) for x in f], dtype=object) for f in cols]
    n = len(cols[0])
    if n == 0:
        return np.zeros(0, dtype=np.uint64)
    lv, ar, od = cols[:3]
    if (tiebreak is None and min(lv) >= 0 and max(lv) <= 7 and min(ar) >= 0
            and max(ar) < (1 << _ARRIVAL_BITS) and min(od) >= 0 and max(od) < (1 << _ORDER_BITS)):
        return ((lv.astype(np.uint64) << np.uint64(61)) | (ar.astype(np.uint64) << np.uint64(_ORDER_BITS))
                | od.astype(np.uint64))
    fields, bits = [], []
    for f in cols:
        uniq = sorted(set(f.tolist()))
        rank = {v: i for i, v in enumerate(uniq)}
        fields.append(np.asarray([rank[v] for v in f.tolist()], dtype=np.uint64))
        bits.append(max(1, (len(uniq) - 1).bit_length()))
    if sum(bits) > 64:
        raise ValueError("queue snapshot too large for 64-bit difficulty keys")
    key = np.zeros(n, dtype=np.uint64)
    for f, b in zip(fields, bits):
        key = (key << np.uint64(b)) | f
    return key


def device_sort(keys: np.ndarray, device="cuda") -> list:
    """Permutation sorting uint64 keys ascending (equal keys keep input order),
    on the GPU: one CTA's shared-memory bitonic sort up to SEGMENT_MAX keys
    (duchess_sort_difficulty), else 4096-key tiles plus merge-path merge
    passes (duchess_sort_keys)."""
    import torch

    from . import _lib
    n = len(keys)
    if n == 0:
        return []
    lib = _lib.load()
    _lib.require_cuda()
    k = torch.from_numpy(np.ascontiguousarray(keys, dtype=np.uint64).view(np.int64)).to(device)
    perm = torch.empty(n, dtype=torch.int32, device=device)
    if n <= SEGMENT_MAX:
        off = torch.tensor([0, n], dtype=torch.int32, device=device)
        _lib.check(lib.duchess_sort_difficulty(k.data_ptr(), off.data_ptr(), 1, perm.data_ptr(),
                                               _lib.stream_handle()), "duchess_sort_difficulty")
    else:
        ws = torch.empty(int(lib.duchess_sort_keys_workspace_bytes(n)), dtype=torch.uint8,
                         device=device)
        _lib.check(lib.duchess_sort_keys(k.data_ptr(), n, perm.data_ptr(), ws.data_ptr(),
                                         ws.numel(), _lib.stream_handle()), "duchess_sort_keys")
    return [int(x) for x in perm.cpu().numpy()]


def difficulty_queue(levels, arrivals=None, device="cuda") -> list:
    """Easiest-first service order of a queue snapshot (level, arrival, order)."""
    n = len(levels)
    arrivals = list(range(n)) if arrivals is None else arrivals
    return device_sort(pack_keys([1 if lv is None else lv for lv in levels], arrivals,
                                 range(n)), device=device)


def next_request(queue: list, policy: str, now: int) -> QueueEntry:
    """Pop the next request to serve (scheduler.py:60-96)."""
    if policy not in SCHEDULES:
        raise ValueError(f"unknown schedule policy {policy!r}")
    idx, lv, ar, od = [], [], [], []
    for i, e in enumerate(queue):
        if e.arrival > now:
            continue
        if policy == FCFS:
            level = 0
        elif policy == EASIEST_ACTUAL:
            if e.trace.difficulty is None:
                raise ValueError(f"request {e.trace.id!r} has no difficulty label; "
                                 f"easiest-actual needs labeled traces")
            level = e.trace.difficulty
        else:
            if e.prefill_done is None or e.prefill_done > now:
                continue
            if e.predicted_difficulty is None:
                raise ValueError(f"request {e.trace.id!r} has no predicted difficulty; "
                                 f"prefill must run before easiest-predicted selection")
            level = e.predicted_difficulty
        idx.append(i)
        lv.append(level)
        ar.append(e.arrival)
        od.append(e.order)
    if not idx:
        raise ValueError("no eligible request")
    # equal (level, arrival, order) tuples: the reference keeps the first in
    # queue order (strict `<`); the bitonic sort is not stable, so the queue
    # position becomes a last key field
    dup = len(set(zip(lv, ar, od))) < len(idx)
    first = device_sort(pack_keys(lv, ar, od, tiebreak=range(len(idx)) if dup else None))[0]
    return queue.pop(idx[first])
