"""CPU restatement of the in-the-round paged KV cache (K3, duchess_kv_round).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): the checker for
paper_2509_24957_b200/csrc/kv.cu, never the measured or shipped path.

The reference has no KV cache: a fork is pure accounting — the child resumes
the next template at the parent's position and the prefix is not re-charged
(reference pkg/src/branchsim/orchestrator.py:254-268 _spawn(offset_base=
source.position), :378-388; the paper serves it with vLLM prefix caching,
PAPER.md:466). This module restates, per request, what the device does with
that accounting on a paged cache, driven by the ORACLE's own rounds
(oracle/port.py DuchessRequest, pinned to the reference's golden vectors):

* one call before the first round (after phase 1 of round 1) and one after
  every round k, seeing the branches as they are after round k AND phase 1
  of round k+1 (the device's duchess_round decides k and advances k+1 in one
  launch; phase 1 is orchestrator.py:344-355, restated in ``phase1``);
* per call, in this order: (1) round k's branch-outs in action order whose
  child is still active — the child row takes the root's first prefix//bt
  blocks (refcount + 1) and one fresh block for a partial tail; (2) rows of
  branches no longer active release their blocks in (branch id, block index)
  order, a block reaching refcount 0 is pushed on the free stack; (3) active
  branches' rows grow to ceil(position / bt) blocks in (branch id, block)
  order, popping the stack first, then blocks above the high-water mark;
* a request that finished in round k releases its whole arena.

The root of a fork is its source, or — when the source is a child spawned
earlier in the same round (orchestrator.py:384-388 appends children to the
pool) — that child's root; the prefix is the child's (clamped) offset_base
(:263).
"""

from __future__ import annotations

import math

from oracle import port


def phase1(req: port.DuchessRequest) -> dict:
    """{branch_id: (status, position)} after phase 1 of the request's next
    round (orchestrator.py:344-355), without mutating the request."""
    k = req.k
    out = {}
    for b in req.branches:
        pos, st = b.position, b.status
        if st == port.ACTIVE:
            room = min(b.template.natural_length, k.token_cap) - pos
            pos += max(0, min(k.interval_tokens, room))
            if pos >= b.template.natural_length:
                st = port.NATURAL_END
            elif pos >= k.token_cap:
                st = port.CAPPED
        out[b.branch_id] = (st, pos)
    return out


class RequestArena:
    """One request's block arena: P blocks, LIFO free stack + high-water mark."""

    def __init__(self, blocks_per_slot: int, block_tokens: int = 16, max_blocks: int = 1 << 30):
        self.P, self.bt, self.NB = blocks_per_slot, block_tokens, max_blocks
        self.reset()

    def reset(self):
        self.rows: dict[int, list] = {}      # branch id -> block ids
        self.tokens: dict[int, int] = {}     # branch id -> tokens covered
        self.ref = [0] * self.P
        self.stack: list[int] = []
        self.hwm = 0
        self.overflow = 0
        self.tail_jobs: list = []            # (src block, dst block, tokens) of the last call

    def _alloc(self) -> int:
        if self.stack:
            return self.stack.pop()
        if self.hwm < self.P:
            self.hwm += 1
            return self.hwm - 1
        self.overflow += 1
        return -1

    def call(self, forks: list, states: dict) -> None:
        """forks: [(child, root, prefix)] in action order; states: {branch:
        (status, position)} after the round and the next phase 1."""
        bt = self.bt
        self.tail_jobs = []
        for child, root, prefix in forks:
            if states[child][0] != port.ACTIVE:
                continue
            n_full, tail = divmod(prefix, bt)
            src = self.rows.get(root, [])
            row = list(src[:n_full])
            for blk in row:
                if blk >= 0:
                    self.ref[blk] += 1
            if tail:
                blk = self._alloc()
                row.append(blk)
                if blk >= 0:
                    self.ref[blk] = 1
                    self.tail_jobs.append((src[n_full], blk, tail))
            self.rows[child] = row
            self.tokens[child] = prefix
        for b in sorted(self.rows):
            if states.get(b, (None,))[0] == port.ACTIVE:
                continue
            for blk in self.rows[b]:
                if blk >= 0:
                    self.ref[blk] -= 1
                    if self.ref[blk] == 0:
                        self.stack.append(blk)
            del self.rows[b]
            del self.tokens[b]
        for b in sorted(states):
            st, pos = states[b]
            if st != port.ACTIVE:
                continue
            row = self.rows.setdefault(b, [])
            want = math.ceil(pos / bt)
            need = min(want, self.NB)
            self.overflow += want - need
            while len(row) < need:
                blk = self._alloc()
                row.append(blk)
                if blk >= 0:
                    self.ref[blk] = 1
            self.tokens[b] = pos

    def snapshot(self) -> dict:
        """Same shape as PagedKVCache.slot_snapshot (without owner / peak)."""
        return {"rows": {b: (self.tokens[b], list(self.rows[b])) for b in sorted(self.rows)
                         if self.tokens[b] > 0},
                "refcount": self.ref[:self.hwm], "stack": list(self.stack), "hwm": self.hwm}


def round_forks(req: port.DuchessRequest, rnd: port.Round) -> list:
    """(child, root, prefix) of a round's branch-outs, in action order."""
    root = {}
    out = []
    for kind, child, src in rnd.actions:
        if kind != "branch_out":
            continue
        r = root.get(src, src)
        root[child] = r
        out.append((child, r, req.branches[child].offset_base))
    return out


def replay(req: port.DuchessRequest, blocks_per_slot: int, block_tokens: int = 16,
           max_blocks: int = 1 << 30) -> list:
    """Run a fresh oracle request to completion; return the arena snapshot
    after every device call: [after phase 1 of round 1, after round 1, ...].
    The snapshot after the finishing round is the empty (reset) arena."""
    arena = RequestArena(blocks_per_slot, block_tokens, max_blocks)
    arena.call([], phase1(req))
    snaps = [arena.snapshot()]
    while not req.done:
        rnd = req.step()
        if req.done:
            arena.reset()
        else:
            arena.call(round_forks(req, rnd), phase1(req))
        snaps.append(arena.snapshot())
    return snaps


def check_invariants(snap: dict, block_tokens: int = 16) -> None:
    """Size-independent properties of one arena snapshot: refcount[b] equals
    the number of rows referencing b; the free stack and the referenced blocks
    partition [0, hwm); every row covers ceil(tokens / bt) blocks, none -1."""
    refs = [0] * snap["hwm"]
    for _b, (tokens, row) in snap["rows"].items():
        assert len(row) == math.ceil(tokens / block_tokens), (tokens, row)
        for blk in row:
            assert 0 <= blk < snap["hwm"], blk
            refs[blk] += 1
    assert refs == list(snap["refcount"]), (refs, snap["refcount"])
    free = sorted(snap["stack"])
    assert len(set(free)) == len(free)
    used = {b for b, n in enumerate(refs) if n}
    assert not used & set(free)
    assert used | set(free) == set(range(snap["hwm"]))
