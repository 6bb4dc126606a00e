"""Paged KV block table with copy-on-write branch-out (K3, ``duchess_fork_cow``).

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
