"""Parity at BASELINE.json's full sizes through size-independent properties.

* C2 scoring: all 4096 windows of a 1 GiB slab (256 requests x 16 branches,
  T=32, H=4096 bf16) scored through the survivor-list path; a random sample of
  windows matches the fp64 oracle within the north-star tolerance and a second
  launch is bit-identical (deterministic reductions).
* C4 fork: the full 24 576-fork trace (512 requests, 16 roots, 48 forks each);
  tables, refcounts and the free cursor equal the serial restatement exactly and
  every private tail holds its root's tail bytes (KV shrunk to 256 B/token so
  the pool stays at 2.3 GB; the copy is length-generic)."""

import numpy as np
import pytest
import torch

from oracle import activations as oact
from oracle import extensions as ext
from oracle import port

pytestmark = pytest.mark.gpu


def test_c2_full_slab_scores_match_oracle_and_repeat_bitwise():
    from paper_2509_24957_b200.probe import ProbeBank, Scorer, fill_windows
    rows, L, T, H = 256 * 16, 1, 32, 4096
    rng = np.random.default_rng(8)
    w = rng.normal(0, 1.5 / np.sqrt(H), (L, H))
    g = rng.uniform(0.5, 1.5, (L, H))
    beta = rng.uniform(-0.1, 0.1, (L, H))
    bank = ProbeBank.from_linear(w, [0.05], g, beta)
    acts = torch.empty((rows, L, T, H), dtype=torch.bfloat16, device="cuda")
    req = torch.arange(rows, dtype=torch.int64, device="cuda") // 16 + 500
    tmpl = torch.arange(rows, dtype=torch.int32, device="cuda") % 16
    pos = (torch.arange(rows, dtype=torch.int32, device="cuda") % 7) * 80 + 80
    fill_windows(acts, 21, req, tmpl, pos)
    lst = torch.arange(rows, dtype=torch.int32, device="cuda")
    cnt = torch.tensor([rows], dtype=torch.int32, device="cuda")
    sc = Scorer(bank, rows * L)
    out = []
    for _ in range(2):
        lg = torch.empty((rows, L), device="cuda")
        pr = torch.empty((rows, L), dtype=torch.float64, device="cuda")
        sc.score_list(acts, lg, pr, lst, cnt)
        out.append(lg.cpu().numpy())
    assert np.array_equal(out[0], out[1])
    reqs, tms, poss = req.cpu().numpy(), tmpl.cpu().numpy(), pos.cpu().numpy()
    for r in np.random.default_rng(1).choice(rows, 48, replace=False):
        win = oact.synth_window(21, int(reqs[r]), int(tms[r]), int(poss[r]), 0, T, H, True)
        ref, _ = port.pooled_linear_probe(win, w[0], 0.05, g[0], beta[0])
        assert abs(float(out[0][r, 0]) - ref) <= 1e-4 * max(abs(ref), 1.0), r


def test_c4_full_trace_tables_refcounts_cursor_and_tails():
    import bench
    from paper_2509_24957_b200.kvfork import BlockTable
    R, roots, nf, bt, max_blocks, kvb = 512, 16, 48, 16, 256, 256
    pos, forks = bench.make_fork_trace(R, roots, nf, bt, max_blocks, seed=31)
    rows_per = roots + nf
    nblk_root = -(-pos // bt)
    n_root_blocks = int(nblk_root.sum())
    n_tail = int(((forks[:, :, 3] % bt) != 0).sum())
    n_blocks = n_root_blocks + n_tail
    table = np.full((R * rows_per, max_blocks), -1, dtype=np.int32)
    nxt = 0
    for r in range(R):
        for b in range(roots):
            table[r * rows_per + b, :nblk_root[r, b]] = np.arange(nxt, nxt + nblk_root[r, b])
            nxt += nblk_root[r, b]
    ref0 = np.zeros(n_blocks, dtype=np.int32)
    ref0[:n_root_blocks] = 1
    free = np.arange(n_root_blocks, n_blocks, dtype=np.int32)
    t = BlockTable(R * rows_per, max_blocks, n_blocks, bt, kvb)
    t.table.copy_(torch.from_numpy(table))
    t.refcount.copy_(torch.from_numpy(ref0))
    t.free_list = torch.from_numpy(free).cuda()
    gen = torch.Generator(device="cuda").manual_seed(5)
    t.kv.copy_(torch.randint(0, 256, t.kv.shape, dtype=torch.uint8, device="cuda", generator=gen))
    kv0 = t.kv.view(n_blocks, bt * kvb).clone()
    t.cursor.zero_()
    t.fork(torch.from_numpy(forks).cuda(), None, 1, rows_per)
    torch.cuda.synchronize()
    wt, wr, wc, _, status = ext.cow_fork_ref(forks, None, table, ref0, free, 0, None, kvb, bt,
                                             rows_per)
    assert status == 0
    got_table = t.table.cpu().numpy()
    assert np.array_equal(got_table, wt)
    assert np.array_equal(t.refcount.cpu().numpy(), wr)
    assert int(t.cursor) == wc == n_tail
    # every private tail block holds its root's first (prefix % 16) tokens
    kv = t.kv.view(n_blocks, bt * kvb)
    g_idx, k_idx = np.nonzero(forks[:, :, 3] % bt)
    child, root, prefix = (forks[g_idx, k_idx, i] for i in (0, 2, 3))
    n_full, tail = prefix // bt, prefix % bt
    dst_blk = got_table[g_idx * rows_per + child, n_full]
    src_blk = table[g_idx * rows_per + root, n_full]
    for tl in range(1, bt):
        sel = tail == tl
        if not sel.any():
            continue
        d = torch.from_numpy(dst_blk[sel].astype(np.int64)).cuda()
        s = torch.from_numpy(src_blk[sel].astype(np.int64)).cuda()
        assert torch.equal(kv[d, :tl * kvb], kv0[s, :tl * kvb]), tl


def test_c5_full_shard_gradient_matches_fp64():
    """K4 over the full per-GPU C5 shard (524 288 x 8192 bf16, 8 GiB) against a
    plain PyTorch fp64 reference computed chunk by chunk on the device."""
    from paper_2509_24957_b200.train import LogisticProbeTrainer
    N, H = 524288, 8192
    g = torch.Generator(device="cuda").manual_seed(5)
    X = torch.empty((N, H), dtype=torch.bfloat16, device="cuda")
    for lo in range(0, N, 65536):
        X[lo:lo + 65536] = torch.randn((65536, H), generator=g, device="cuda").to(torch.bfloat16)
    w_true = torch.randn(H, generator=g, device="cuda") / np.sqrt(H)
    y = torch.empty(N, device="cuda")
    for lo in range(0, N, 65536):
        p = torch.sigmoid(X[lo:lo + 65536].float() @ w_true)
        y[lo:lo + 65536] = (torch.rand(65536, generator=g, device="cuda") < p).float()
    tr = LogisticProbeTrainer(H)
    tr.w.copy_(torch.randn(H + 1, generator=g, device="cuda") / np.sqrt(H))
    got = tr.local_grad(X, y, 1.0 / N).double()
    w64 = tr.w.double()
    ref = torch.zeros(H + 1, dtype=torch.float64, device="cuda")
    for lo in range(0, N, 32768):
        xc = X[lo:lo + 32768].double()
        r = torch.sigmoid(xc @ w64[:H] + w64[H]) - y[lo:lo + 32768].double()
        ref[:H] += xc.T @ r
        ref[H] += r.sum()
    ref /= N
    torch.testing.assert_close(got, ref, rtol=1e-4, atol=1e-4 * float(ref.abs().max()))


def test_c2_engine_scale_decisions_match_oracle():
    """K2 at the C2 engine size: 256 request slots x 16 branches with the
    math-like knobs over a 1024-request pool (64 templates each, easiest-first
    queue, on-device refill) — every request's RoundReports and outcome equal
    the oracle's (trace / synthetic predictor, rho 0.8)."""
    import random
    from paper_2509_24957_b200 import _lib
    from paper_2509_24957_b200.engine import BatchedDuchess
    from paper_2509_24957_b200.scheduler import difficulty_queue
    from tests.golden_util import port_report_tuple
    import bench
    knobs = port.Knobs(max_branches=16, **bench.PRESET_KNOBS["math-like"])
    params = port.GenParams(templates_per_request=64, **bench.PRESET_GEN["math-like"])
    traces = port.generate(params, 1024, seed=17)
    master = random.Random(18)
    seeds = [master.getrandbits(64) for _ in traces]
    queue = difficulty_queue([t.difficulty for t in traces])
    eng = BatchedDuchess(traces, knobs, seeds, n_slots=256, pred_source=_lib.PRED_TRACE,
                         rho=0.8, queue=queue)
    eng.advance()
    reports = {}
    for _ in range(100000):
        eng.round()
        for p, rep in eng.round_reports():
            reports.setdefault(p, []).append(rep)
        if eng.all_done():
            break
    assert eng.all_done()
    assert int(eng.counters()[_lib.CNT_AMBIGUOUS]) == 0
    outcomes = eng.outcomes()
    for p, tr in enumerate(traces):
        ref = port.DuchessRequest(tr, knobs, random.Random(seeds[p]), rho=0.8)
        want = []
        while not ref.done:
            want.append(port_report_tuple(ref.step()))
        assert reports[p] == want, f"request {p}"
        o = ref.outcome
        assert (outcomes[p]["final"], outcomes[p]["reason"], outcomes[p]["tally"],
                outcomes[p]["tokens_decode"], outcomes[p]["rounds"]) == (
            o.final, o.termination_reason, o.tally, o.tokens_decode, o.rounds)
