"""The paged-KV restatement (oracle/kvcache.py) on the CPU: a hand-computed
known answer for one call sequence, and size-independent properties of
arenas replayed from the oracle's own rounds (which are pinned to the
reference's golden vectors, tests/test_oracle_golden.py)."""

import random

import pytest

from oracle import kvcache, port
from tests.golden_util import case_knobs, case_traces, load

A, E = port.ACTIVE, port.EARLY_TERMINATED


def test_arena_known_answer():
    ar = kvcache.RequestArena(blocks_per_slot=16, block_tokens=16)
    ar.call([], {0: (A, 20), 1: (A, 20)})
    assert ar.snapshot() == {"rows": {0: (20, [0, 1]), 1: (20, [2, 3])},
                             "refcount": [1, 1, 1, 1], "stack": [], "hwm": 4}
    # branch 2 forks from 0 at 20 tokens (1 shared block + a copied 4-token
    # tail); branch 1 early-terminates; 0 and 2 decode to 36 tokens
    ar.call([(2, 0, 20)], {0: (A, 36), 1: (E, 20), 2: (A, 36)})
    assert ar.tail_jobs == [(1, 4, 4)]
    assert ar.snapshot() == {"rows": {0: (36, [0, 1, 3]), 2: (36, [0, 4, 2])},
                             "refcount": [2, 1, 1, 1, 1], "stack": [], "hwm": 5}
    # a fork on a block boundary shares every block, no tail
    ar.call([(3, 2, 32)], {0: (E, 36), 1: (E, 20), 2: (A, 52), 3: (A, 48)})
    assert ar.tail_jobs == []
    snap = ar.snapshot()
    assert snap["rows"] == {2: (52, [0, 4, 2, 3]), 3: (48, [0, 4, 1])}
    assert snap["stack"] == []
    kvcache.check_invariants(snap)


def test_arena_overflow_counts():
    ar = kvcache.RequestArena(blocks_per_slot=2, block_tokens=16)
    ar.call([], {0: (A, 40)})
    assert ar.overflow == 1 and ar.rows[0] == [0, 1, -1]


def _replays(case, P=4096):
    traces = case_traces(case)
    knobs = case_knobs(case)
    for t, r in zip(traces, case["requests"]):
        req = port.DuchessRequest(t, knobs, random.Random(int(r["seed"])), rho=case["rho"])
        yield kvcache.replay(req, P)


@pytest.mark.parametrize("case", load("decisions.json"), ids=lambda c: c["name"])
def test_replayed_arenas_keep_invariants(case):
    for snaps in _replays(case):
        for s in snaps:
            kvcache.check_invariants(s)
        assert snaps[-1] == {"rows": {}, "refcount": [], "stack": [], "hwm": 0}


def test_replay_is_deterministic_and_shares_prefixes():
    case = load("decisions.json")[0]
    a = [s for snaps in _replays(case) for s in snaps]
    b = [s for snaps in _replays(case) for s in snaps]
    assert a == b
    shared = sum(1 for s in a for n in s["refcount"] if n > 1)
    assert shared > 0, "no block was ever shared by a fork"
