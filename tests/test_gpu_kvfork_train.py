"""K3 (copy-on-write block-table fork) and K4 (logistic-regression gradient)
parity against the CPU restatements in oracle/extensions.py."""

import random

import numpy as np
import pytest
import torch

from oracle import extensions as ext
from tests.golden_util import case_knobs, case_traces, load

pytestmark = pytest.mark.gpu


def _random_tables(rng, n_groups, rows_per_group, stride, n_roots, bt, n_blocks_free):
    """Root branches with allocated block rows; returns table, refcount, free list,
    root positions (dict (g, id) -> tokens)."""
    rows = n_groups * rows_per_group
    table = np.full((rows, stride), -1, dtype=np.int32)
    next_blk = 0
    positions = {}
    for g in range(n_groups):
        for b in range(n_roots):
            pos = rng.randint(0, stride * bt)
            nblk = -(-pos // bt)
            table[g * rows_per_group + b, :nblk] = np.arange(next_blk, next_blk + nblk)
            next_blk += nblk
            positions[(g, b)] = pos
    n_blocks = next_blk + n_blocks_free
    refcount = np.zeros(n_blocks, dtype=np.int32)
    refcount[:next_blk] = 1
    free_list = np.arange(next_blk, n_blocks, dtype=np.int32)
    return table, refcount, free_list, positions, n_blocks


@pytest.mark.parametrize("seed,kv_bpt,free_extra", [(0, 64, 400), (1, 0, 400), (2, 48, 5)])
def test_fork_cow_matches_serial_restatement(seed, kv_bpt, free_extra):
    from paper_2509_24957_b200.kvfork import BlockTable
    rng = random.Random(seed)
    n_groups, rows_per_group, stride, bt, n_roots, cap = 6, 40, 24, 16, 8, 12
    table, refcount, free_list, positions, n_blocks = _random_tables(
        rng, n_groups, rows_per_group, stride, n_roots, bt, free_extra)
    forks = np.zeros((n_groups, cap, 4), dtype=np.int32)
    counts = np.zeros(n_groups, dtype=np.int32)
    for g in range(n_groups):
        n = rng.randint(0, cap)
        counts[g] = n
        for k in range(n):
            root = rng.randrange(n_roots)
            prefix = rng.randint(0, positions[(g, root)])
            forks[g, k] = (n_roots + k, root, root, prefix)
    bt_dev = BlockTable(n_groups * rows_per_group, stride, n_blocks, bt, kv_bpt)
    bt_dev.table.copy_(torch.from_numpy(table))
    bt_dev.refcount.copy_(torch.from_numpy(refcount))
    bt_dev.free_list = torch.from_numpy(free_list).cuda()
    kv = None
    if kv_bpt:
        kv = np.frombuffer(np.random.default_rng(seed).bytes(bt_dev.kv.numel()), dtype=np.uint8).copy()
        bt_dev.kv.copy_(torch.from_numpy(kv))
    bt_dev.fork(torch.from_numpy(forks).cuda(), torch.from_numpy(counts).cuda(), 1,
                rows_per_group)
    torch.cuda.synchronize()
    want_t, want_r, want_c, want_kv, want_s = ext.cow_fork_ref(
        forks, counts, table, refcount, free_list, 0, kv, kv_bpt, bt, rows_per_group)
    assert np.array_equal(bt_dev.table.cpu().numpy(), want_t)
    assert np.array_equal(bt_dev.refcount.cpu().numpy(), want_r)
    assert int(bt_dev.cursor) == want_c
    assert int(bt_dev.status) == want_s
    if kv_bpt:
        assert np.array_equal(bt_dev.kv.cpu().numpy(), want_kv)


def test_engine_fork_records_drive_cow_fork():
    """Fork records emitted by duchess_decide (chains pre-resolved to the
    table root) applied by K3 == serial restatement, round after round."""
    from paper_2509_24957_b200 import _lib
    from paper_2509_24957_b200.engine import BatchedDuchess
    from paper_2509_24957_b200.kvfork import BlockTable
    case = next(c for c in load("decisions.json") if c["name"] == "math_c16")
    traces = case_traces(case)
    eng = BatchedDuchess(traces, case_knobs(case), [int(r["seed"]) for r in case["requests"]],
                         n_slots=len(traces), pred_source=_lib.PRED_TRACE, rho=case["rho"])
    R, C, B = eng.R, eng.C, eng.wl.branch_cap
    stride, bt_tokens = 128, 16
    rng = random.Random(3)
    n_checked = 0
    for _ in range(60):
        eng.step()
        rec = eng.t["round_rec"].view(R, _lib.REC_WORDS).cpu().numpy()
        nf = rec[:, _lib.REC_NFORKS].astype(np.int32)
        if nf.sum() == 0:
            if eng.all_done():
                break
            continue
        forks = eng.t["forks"].view(R, C, 4).cpu().numpy()
        # synthetic tables for every root referenced this round
        table = np.full((R * B, stride), -1, dtype=np.int32)
        need = {}
        for r in range(R):
            for k in range(nf[r]):
                child, src, root, prefix = forks[r, k]
                assert prefix >= 0
                need[r * B + root] = max(need.get(r * B + root, 0), int(prefix))
        nxt = 0
        for row, prefix in sorted(need.items()):
            nblk = -(-rng.randint(prefix, prefix + 40) // bt_tokens)
            table[row, :nblk] = np.arange(nxt, nxt + nblk)
            nxt += nblk
        n_blocks = nxt + 64 * C
        ref = np.ones(n_blocks, dtype=np.int32)
        ref[nxt:] = 0
        free = np.arange(nxt, n_blocks, dtype=np.int32)
        dev = BlockTable(R * B, stride, n_blocks, bt_tokens, 32)
        dev.table.copy_(torch.from_numpy(table))
        dev.refcount.copy_(torch.from_numpy(ref))
        dev.free_list = torch.from_numpy(free).cuda()
        kv = np.frombuffer(np.random.default_rng(n_checked).bytes(dev.kv.numel()),
                           dtype=np.uint8).copy()
        dev.kv.copy_(torch.from_numpy(kv))
        dev.fork_from_engine(eng)
        torch.cuda.synchronize()
        wt, wr, wc, wkv, _ = ext.cow_fork_ref(forks, nf, table, ref, free, 0, kv, 32,
                                              bt_tokens, B)
        assert np.array_equal(dev.table.cpu().numpy(), wt)
        assert np.array_equal(dev.refcount.cpu().numpy(), wr)
        assert int(dev.cursor) == wc
        assert np.array_equal(dev.kv.cpu().numpy(), wkv)
        n_checked += 1
        if eng.all_done():
            break
    assert n_checked > 3


@pytest.mark.parametrize("dtype,N,H", [(torch.bfloat16, 3000, 1024), (torch.float32, 777, 512),
                                       (torch.bfloat16, 5, 8192), (torch.bfloat16, 40000, 256),
                                       # C5 row width, stage kept in registers, ragged last stage
                                       (torch.bfloat16, 2999, 8192), (torch.float32, 1001, 8192),
                                       # rows too wide to keep: two-CTA re-read kernel
                                       (torch.bfloat16, 613, 16384),
                                       # partial last vector column block
                                       (torch.bfloat16, 1234, 5128)])
def test_lr_grad_matches_fp64(dtype, N, H):
    from paper_2509_24957_b200.train import LogisticProbeTrainer
    g = torch.Generator(device="cuda").manual_seed(N + H)
    X = torch.randn((N, H), generator=g, device="cuda").to(dtype)
    w = torch.randn(H + 1, generator=g, device="cuda") / np.sqrt(H)
    y = (torch.rand(N, generator=g, device="cuda") < 0.4).float()
    tr = LogisticProbeTrainer(H)
    tr.w.copy_(w)
    got = tr.local_grad(X, y, 1.0 / N).cpu().numpy()
    ref = ext.lr_grad_ref(X.float().cpu().numpy(), y.cpu().numpy(), w.cpu().numpy())
    np.testing.assert_allclose(got, ref, rtol=1e-4, atol=1e-4 * np.abs(ref).max())


def test_sharded_gradients_sum_to_full_gradient():
    """Data-parallel decomposition used by the NCCL path: per-shard partial
    gradients (scaled by 1/N_total) sum to the full-batch gradient."""
    from paper_2509_24957_b200.train import LogisticProbeTrainer, shard_rows
    N, H, world = 10001, 768, 4
    g = torch.Generator(device="cuda").manual_seed(7)
    X = torch.randn((N, H), generator=g, device="cuda").to(torch.bfloat16)
    y = (torch.rand(N, generator=g, device="cuda") < 0.5).float()
    tr = LogisticProbeTrainer(H)
    tr.w.copy_(torch.randn(H + 1, generator=g, device="cuda") / 30)
    full = tr.local_grad(X, y, 1.0 / N).clone()
    parts = torch.zeros_like(full)
    for rank in range(world):
        lo, hi = shard_rows(N, rank, world)
        parts += tr.local_grad(X[lo:hi].contiguous(), y[lo:hi].contiguous(), 1.0 / N)
    torch.testing.assert_close(parts, full, rtol=1e-5, atol=1e-6)


def test_training_reduces_loss():
    from paper_2509_24957_b200.train import LogisticProbeTrainer
    N, H = 20000, 512
    g = torch.Generator(device="cuda").manual_seed(1)
    X = torch.randn((N, H), generator=g, device="cuda").to(torch.bfloat16)
    w_true = torch.randn(H, generator=g, device="cuda") / np.sqrt(H) * 3
    y = (torch.rand(N, generator=g, device="cuda") < torch.sigmoid(X.float() @ w_true)).float()
    tr = LogisticProbeTrainer(H, lr=2.0)

    def loss():
        z = X.float() @ tr.w[:-1] + tr.w[-1]
        return torch.nn.functional.binary_cross_entropy_with_logits(z, y).item()
    l0 = loss()
    for _ in range(30):
        tr.step(X, y, N)
    assert loss() < l0 - 0.05
