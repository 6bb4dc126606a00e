"""Edge cases through the C-ABI on the GPU: empty launches, the > 64-answer
tally path, the widest rows the TMA scorer takes, requests with a single
template, and the score-list path over an empty survivor list."""

import random

import numpy as np
import pytest
import torch

from oracle import activations as oact
from oracle import port
from tests.golden_util import port_report_tuple

pytestmark = pytest.mark.gpu


def test_empty_launches_are_no_ops():
    from paper_2509_24957_b200 import _lib
    lib = _lib.load()
    s = _lib.stream_handle()
    x = torch.zeros(64, dtype=torch.bfloat16, device="cuda")
    f = torch.zeros(64, dtype=torch.float32, device="cuda")
    d = torch.zeros(64, dtype=torch.float64, device="cuda")
    i = torch.zeros(64, dtype=torch.int32, device="cuda")
    assert lib.duchess_score(x.data_ptr(), _lib.BF16, 0, 1, 1, 8, 8, 8, 8, f.data_ptr(),
                             f.data_ptr(), None, f.data_ptr(), d.data_ptr(), None, 0, 0, 0,
                             s) == 0
    assert lib.duchess_sort_difficulty(i.data_ptr(), i.data_ptr(), 0, i.data_ptr(), s) == 0
    assert lib.duchess_vote(i.data_ptr(), 0, 4, 1, 1, i.data_ptr(), i.data_ptr(), s) == 0
    assert lib.duchess_timeline(i.data_ptr(), 0, 25.0, 0.0, 0, i.data_ptr(), i.data_ptr(), s) == 0
    assert lib.duchess_confused_levels(i.data_ptr(), 0, i.data_ptr(), d.data_ptr(),
                                       i.data_ptr(), s) == 0
    assert lib.duchess_tc_linear(x.data_ptr(), 0, 64, x.data_ptr(), 256, 0, None, f.data_ptr(),
                                 f.data_ptr(), f.data_ptr(), 0, x.data_ptr(), None, 0, s) == 0
    torch.cuda.synchronize()


def test_score_active_with_no_survivors_writes_nothing():
    from paper_2509_24957_b200 import _lib
    from paper_2509_24957_b200.engine import BatchedDuchess
    from paper_2509_24957_b200.probe import ProbeBank, Scorer
    knobs = port.Knobs(max_branches=4, interval_tokens=16)
    tr = port.Trace("t", "7", 0, [port.Tmpl(16, "7")])
    eng = BatchedDuchess([tr], knobs, [1], n_slots=2, pred_source=_lib.PRED_DEVICE)
    eng.advance()                            # the only branch ends naturally: no survivor
    assert int(eng.t["active_count"][0]) == 0
    H = 64
    bank = ProbeBank.from_linear(np.ones((1, H)) / H, [0.0])
    acts = torch.zeros((2 * 4, 1, 2, H), dtype=torch.bfloat16, device="cuda")
    logit = torch.full((8, 1), 7.0, device="cuda")
    prob = torch.full((8, 1), 7.0, dtype=torch.float64, device="cuda")
    Scorer(bank, 8).score_active(acts, logit, prob, eng)
    torch.cuda.synchronize()
    assert (logit == 7.0).all() and (prob == 7.0).all()


def _many_answer_traces(n_req, n_ans, seed):
    """Requests whose templates carry > 64 distinct answers (final + probes), so
    the device tally takes its general (non-register) path."""
    rng = random.Random(seed)
    out = []
    for r in range(n_req):
        tm = []
        for j in range(n_ans):
            nat = rng.randint(40, 200)
            probes = [(16 * k, f"a{rng.randrange(n_ans * 2)}") for k in range(1, nat // 16 + 1)]
            tm.append(port.Tmpl(nat, f"a{j}", probes, rng.choice([None, nat // 2])))
        out.append(port.Trace(f"r{r}", "a0", 10, tm, 1 + r % 5))
    return out


def test_more_than_64_answers_matches_oracle():
    from paper_2509_24957_b200 import _lib
    from paper_2509_24957_b200.engine import BatchedDuchess
    traces = _many_answer_traces(6, 90, 3)
    knobs = port.Knobs(max_branches=16, interval_tokens=16, early_term_threshold=0.6,
                       early_term_rounds=1, consensus_frac=1.0, coverage_frac=1.0)
    seeds = [11 + k for k in range(len(traces))]
    eng = BatchedDuchess(traces, knobs, seeds, n_slots=3, pred_source=_lib.PRED_TRACE, rho=0.5)
    assert eng.wl.answer_cap > 64
    reports = {}
    for _ in range(10000):
        eng.step()
        for p, rep in eng.round_reports():
            reports.setdefault(p, []).append(rep)
        if eng.all_done():
            break
    outcomes = eng.outcomes()
    for p, tr in enumerate(traces):
        ref = port.DuchessRequest(tr, knobs, random.Random(seeds[p]), rho=0.5)
        want = []
        while not ref.done:
            want.append(port_report_tuple(ref.step()))
        assert reports[p] == want, f"request {p}"
        assert outcomes[p]["tally"] == ref.outcome.tally
        assert outcomes[p]["final"] == ref.outcome.final


def test_widest_tma_rows_match_oracle():
    """H = 16384 bf16 (32 KB rows, one token per TMA stage, 8 vectors per
    consumer thread) through the list path."""
    from paper_2509_24957_b200.probe import ProbeBank, Scorer, fill_windows
    rows, L, T, H = 6, 1, 3, 16384
    rng = np.random.default_rng(5)
    w = rng.normal(0, 1.5 / np.sqrt(H), (1, H))
    g = rng.uniform(0.5, 1.5, (1, H))
    beta = rng.uniform(-0.1, 0.1, (1, H))
    bank = ProbeBank.from_linear(w, [0.1], g, beta)
    acts = torch.empty((rows, L, T, H), dtype=torch.bfloat16, device="cuda")
    req = torch.arange(rows, dtype=torch.int64, device="cuda") + 40
    tmpl = torch.zeros(rows, dtype=torch.int32, device="cuda")
    pos = torch.arange(rows, dtype=torch.int32, device="cuda") * 16
    fill_windows(acts, 9, req, tmpl, pos)
    lst = torch.tensor([4, 1, 5], dtype=torch.int32, device="cuda")
    cnt = torch.tensor([3], dtype=torch.int32, device="cuda")
    logit = torch.zeros((rows, L), device="cuda")
    prob = torch.zeros((rows, L), dtype=torch.float64, device="cuda")
    Scorer(bank, rows * L).score_list(acts, logit, prob, lst, cnt)
    torch.cuda.synchronize()
    for r in range(rows):
        if r not in (4, 1, 5):
            assert float(logit[r, 0]) == 0.0
            continue
        win = oact.synth_window(9, 40 + r, 0, 16 * r, 0, T, H, True)
        ref, _ = port.pooled_linear_probe(win, w[0], 0.1, g[0], beta[0])
        assert abs(float(logit[r, 0]) - ref) <= 1e-4 * max(abs(ref), 1.0)


def test_device_mt_seeding_matches_cpython():
    """duchess_mt_seed == random.Random(seed).getstate() after its pending
    twist (engine.pretwist), for seeds of one and two 32-bit words."""
    from paper_2509_24957_b200.engine import mt_state_words, pretwist, seed_states
    rng = random.Random(7)
    seeds = [0, 1, 12345, 2 ** 32 - 1, 2 ** 32, 2 ** 64 - 1] + [rng.getrandbits(64) for _ in range(50)]
    got = seed_states(seeds).cpu().numpy().view(np.uint32).reshape(len(seeds), 625)
    for s, row in zip(seeds, got):
        assert np.array_equal(row, pretwist(mt_state_words(s))), s
        r = random.Random(s)
        a = [r.random() for _ in range(3)]
        r2 = random.Random()
        r2.setstate((3, tuple(int(x) for x in row), None))
        assert [r2.random() for _ in range(3)] == a


def test_upload_survivors_rejects_pageable_host_memory():
    from paper_2509_24957_b200 import _lib
    lib = _lib.load()
    host = torch.zeros(1024, dtype=torch.uint8)                  # pageable
    dev = torch.zeros(1024, dtype=torch.uint8, device="cuda")
    rows = torch.zeros(4, dtype=torch.int32, device="cuda")
    cnt = torch.zeros(4, dtype=torch.int32, device="cuda")
    assert lib.duchess_gather_active(host.data_ptr(), dev.data_ptr(), 256, rows.data_ptr(),
                                     cnt.data_ptr(), 4, _lib.stream_handle()) == 1


def test_launch_gate_holds_the_stream_until_released_or_timeout():
    """bench.py's measurement gate (duchess_gate): work queued behind it does
    not run until the host writes the pinned flag; without the write it gives
    up after its timeout and reports that."""
    import time

    from paper_2509_24957_b200 import _lib
    lib = _lib.load()
    st = torch.cuda.current_stream()
    flag = torch.zeros(1, dtype=torch.int32).pin_memory()
    timed_out = torch.zeros(1, dtype=torch.int32, device="cuda")
    x = torch.zeros(1, device="cuda")
    x.add_(0)          # load the add kernel now: a first (lazy) module load would wait for the gate
    torch.cuda.synchronize()
    _lib.check(lib.duchess_gate(flag.data_ptr(), 5_000_000_000, timed_out.data_ptr(),
                                st.cuda_stream), "gate")
    x.add_(1)
    time.sleep(0.05)
    assert not st.query()                        # held
    flag.fill_(1)
    torch.cuda.synchronize()
    assert float(x.item()) == 1.0 and int(timed_out.item()) == 0
    flag.zero_()
    _lib.check(lib.duchess_gate(flag.data_ptr(), 20_000_000, timed_out.data_ptr(),
                                st.cuda_stream), "gate")
    torch.cuda.synchronize()                     # released by the 20 ms timeout
    assert int(timed_out.item()) == 1
