"""Paged KV block tables with copy-on-write branch-out (K3).

``PagedKVCache`` (``duchess_kv_round``) is the in-the-round path: a persistent
paged KV cache that follows an engine's rounds — the round's forks share the
root's full blocks and copy its partial tail, ended / cancelled branches
release their blocks, decoding branches grow — with one block arena per
request slot. ``BlockTable`` (``duchess_fork_cow``) applies a batch of fork
records to a flat table (the C4 branch-out-heavy trace).

The reference's fork is ``_spawn(offset_base=source.position)``
(orchestrator.py:254-268): the child resumes at the parent's position and the
prefix is not recomputed. On a paged KV cache that is a block-table
duplication: the child shares the root's full blocks (refcount += 1) and gets
a private copy of the partial tail block. ``BlockTable.fork`` consumes fork
records exactly as ``duchess_decide`` emits them (DuchessState.forks, one
group per request slot) or any flat list.
"""

from __future__ import annotations

import torch

from . import _lib


class BlockTable:
    def __init__(self, n_rows: int, max_blocks: int, n_blocks: int, block_tokens: int = 16,
                 kv_bytes_per_token: int = 0, device="cuda"):
        _lib.require_cuda()
        self.lib = _lib.load()
        self.device = torch.device(device)
        self.block_tokens = block_tokens
        self.kv_bytes_per_token = kv_bytes_per_token
        self.table = torch.full((n_rows, max_blocks), -1, dtype=torch.int32, device=self.device)
        self.refcount = torch.zeros(n_blocks, dtype=torch.int32, device=self.device)
        self.free_list = torch.arange(n_blocks, dtype=torch.int32, device=self.device)
        self.cursor = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.status = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.kv = (torch.zeros(n_blocks * block_tokens * kv_bytes_per_token, dtype=torch.uint8,
                               device=self.device) if kv_bytes_per_token else None)
        self._ws = torch.zeros(16, dtype=torch.uint8, device=self.device)

    def _workspace(self, n_groups: int, group_cap: int) -> torch.Tensor:
        need = int(self.lib.duchess_fork_workspace_bytes(n_groups, group_cap))
        if self._ws.numel() < need:
            self._ws = torch.zeros(need, dtype=torch.uint8, device=self.device)
        return self._ws

    def fork(self, forks: torch.Tensor, group_counts: torch.Tensor | None = None,
             counts_stride: int = 1, rows_per_group: int = 0, stream=None) -> None:
        """forks: int32 [n_groups, group_cap, 4] (child, source, root, prefix)
        on device; group g has group_counts[g * counts_stride] valid records
        (None: all). Branch ids map to table rows g * rows_per_group + id."""
        if forks.dtype != torch.int32 or forks.dim() != 3 or forks.shape[2] != 4:
            raise ValueError("forks must be int32 [n_groups, group_cap, 4]")
        n_groups, cap = forks.shape[0], forks.shape[1]
        ws = self._workspace(n_groups, cap)
        _lib.check(self.lib.duchess_fork_cow(
            forks.data_ptr(), cap, _lib.ptr(group_counts), counts_stride, n_groups,
            rows_per_group, self.table.data_ptr(), self.table.shape[1],
            self.refcount.data_ptr(), self.free_list.data_ptr(), self.free_list.numel(),
            self.cursor.data_ptr(), _lib.ptr(self.kv), self.kv_bytes_per_token,
            self.block_tokens, self.status.data_ptr(), ws.data_ptr(), ws.numel(),
            _lib.stream_handle(stream)), "duchess_fork_cow")

    def fork_from_engine(self, engine, stream=None) -> None:
        """Apply the forks duchess_decide emitted in the latest round (table
        rows = slot * branch_cap + branch id)."""
        R, C = engine.R, engine.C
        forks = engine.t["forks"].view(R, C, 4)
        counts = engine.t["round_rec"][_lib.REC_NFORKS:]
        self.fork(forks, counts, _lib.REC_WORDS, engine.wl.branch_cap, stream)


class PagedKVCache:
    """Persistent paged KV cache of an engine's request slots (K3 in the round).

    engine: BatchedDuchess (its R slots x branch_cap branch ids are the table
    rows). blocks_per_slot: the arena of each slot (default: room for
    max_branches branches at the token cap, i.e. no overflow possible).
    kv_bytes_per_token: KV bytes per token in the pool (0: tables only; one
    Llama-3-8B layer slice is 2*8*128*2 = 4096). Call ``round()`` right after
    every ``engine.round()`` and once after the engine's first ``advance()``.
    """

    def __init__(self, engine, *, block_tokens: int = 16, blocks_per_slot: int | None = None,
                 kv_bytes_per_token: int = 0, max_blocks: int | None = None):
        _lib.require_cuda()
        self.lib = _lib.load()
        self.engine = engine
        dev = engine.device
        self.device = dev
        R, B, C = engine.R, engine.wl.branch_cap, engine.C
        cap = int(engine.policy.token_cap)
        nb = -(-cap // block_tokens) if max_blocks is None else int(max_blocks)
        P = C * nb if blocks_per_slot is None else int(blocks_per_slot)
        if block_tokens < 1 or P < 1 or nb < 1:
            raise ValueError("block_tokens, blocks_per_slot and max_blocks must be positive")
        if R * P >= 2 ** 31:
            raise ValueError("R * blocks_per_slot must fit int32 block ids")
        self.R, self.B, self.C, self.P, self.NB = R, B, C, P, nb
        self.block_tokens, self.kv_bytes_per_token = block_tokens, int(kv_bytes_per_token)
        i32 = dict(dtype=torch.int32, device=dev)
        t = {"table": torch.full((R * B * nb,), -1, **i32),
             "kv_tokens": torch.zeros(R * B, **i32),
             "refcount": torch.zeros(R * P, **i32),
             "free_stack": torch.zeros(R * P, **i32),
             "arena": torch.zeros(R * 4, **i32),
             "jobs": torch.zeros(R * C * 4, **i32),
             "job_count": torch.zeros(R, **i32),
             "counters": torch.zeros(_lib.KV_N_COUNTERS, dtype=torch.int64, device=dev)}
        t["arena"].view(R, 4)[:, 2] = -1
        if kv_bytes_per_token:
            t["kv_pool"] = torch.zeros(R * P * block_tokens * self.kv_bytes_per_token,
                                       dtype=torch.uint8, device=dev)
        self.t = t
        st = _lib.KV()
        st.block_tokens, st.blocks_per_slot, st.max_blocks = block_tokens, P, nb
        st.kv_bytes_per_token = self.kv_bytes_per_token
        for name in _lib.KV_PTR_FIELDS:
            if name in t:
                setattr(st, name, t[name].data_ptr())
        self.struct = st

    def round(self, stream=None, overlap: bool = False, lead: bool = False) -> None:
        """Apply the engine's latest round: forks (with the tail copies of
        their partial blocks), releases, appends. overlap: run beside the
        preceding kernel in the stream (DUCHESS_KV_OVERLAP) — legal right
        after the next round's scorer launch (score(k+1) -> kv(k) ->
        round(k+1)), never after the engine's own round(). lead: right after
        the engine's round(), releasing the next round's scorer at once
        (DUCHESS_KV_LEAD; that scorer must be launched with no_input_wait)."""
        if overlap and lead:
            raise ValueError("overlap and lead are exclusive")
        self.struct.flags = _lib.KV_OVERLAP if overlap else (_lib.KV_LEAD if lead else 0)
        _lib.check(self.lib.duchess_kv_round(self.engine.policy, self.engine.state, self.struct,
                                             _lib.stream_handle(stream)), "duchess_kv_round")

    def counters(self) -> dict:
        c = self.t["counters"].cpu().numpy()
        return {"blocks_allocated": int(c[_lib.KV_CNT_ALLOC]),
                "blocks_released": int(c[_lib.KV_CNT_FREE]),
                "tail_bytes": int(c[_lib.KV_CNT_TAIL_BYTES]),
                "overflow": int(c[_lib.KV_CNT_OVERFLOW])}

    STATE = ("table", "kv_tokens", "refcount", "free_stack", "arena")

    def state_copy(self) -> dict:
        """Device clones of the cache state (stream-ordered, no sync): for
        snapshots taken inside a stream of rounds; see snapshot_of."""
        return {k: self.t[k].clone() for k in self.STATE}

    def slot_snapshot(self, slot: int, state: dict | None = None) -> dict:
        """Host copy of one slot's arena with LOCAL block ids: per branch id
        the table row (blocks covering kv_tokens), refcounts [0, hwm), the free
        stack, hwm, the owning pool index and the peak. state: a state_copy()
        (default: the live state)."""
        t = self.t if state is None else state
        R, B, P, nb, bt = self.R, self.B, self.P, self.NB, self.block_tokens
        ar = t["arena"].view(R, 4)[slot].cpu().numpy()
        top, hwm = int(ar[0]), int(ar[1])
        kvt = t["kv_tokens"].view(R, B)[slot].cpu().numpy()
        tab = t["table"].view(R, B, nb)[slot].cpu().numpy()
        rows = {}
        for b in range(B):
            n = -(-int(kvt[b]) // bt)
            if n:
                rows[b] = (int(kvt[b]), [int(x) - slot * P if x >= 0 else -1 for x in tab[b, :n]])
        ref = t["refcount"].view(R, P)[slot, :hwm].cpu().numpy()
        stack = t["free_stack"].view(R, P)[slot, :top].cpu().numpy()
        return {"rows": rows, "refcount": [int(x) for x in ref], "stack": [int(x) for x in stack],
                "hwm": hwm, "owner": int(ar[2]), "peak": int(ar[3])}
