"""duchess_gather_active (the e2e input path): survivor windows uploaded
from pinned host memory, through the C-ABI."""

import numpy as np
import pytest
import torch

from oracle import port

pytestmark = pytest.mark.gpu


def _setup(n_req, c, temperature, templates=64):
    import random
    knobs = port.Knobs(max_branches=c, interval_tokens=16, early_term_threshold=0.70,
                       early_term_rounds=2, branch_out_temperature=temperature,
                       consensus_frac=0.6, coverage_frac=0.8)
    params = port.GenParams(level_median_tokens=(180, 220, 260, 300, 350),
                            level_correct_prob=(0.92, 0.88, 0.84, 0.80, 0.75),
                            templates_per_request=templates, probe_stride=16)
    traces = port.generate(params, n_req, seed=7)
    master = random.Random(11)
    seeds = [master.getrandbits(64) for _ in traces]
    return knobs, traces, seeds


def test_upload_survivors_copies_only_listed_rows():
    """duchess_gather_active: exactly the rows of the round in flight's active
    list (either parity) arrive from pinned host memory; others untouched."""
    from paper_2509_24957_b200 import _lib
    from paper_2509_24957_b200.engine import BatchedDuchess
    knobs, traces, seeds = _setup(40, 8, 1.0)
    R, C = 6, 8
    eng = BatchedDuchess(traces, knobs, seeds, n_slots=R, pred_source=_lib.PRED_DEVICE,
                         queue=list(range(len(traces))), cycle=True)
    host = torch.randint(-1000, 1000, (R * C, 1, 3, 64), dtype=torch.int16).view(
        torch.bfloat16).pin_memory()
    eng.advance()
    for step in range(6):
        dev = torch.zeros_like(host, device="cuda")
        eng.upload_survivors(host, dev)
        torch.cuda.synchronize()
        mask = eng.t["row_mask"].cpu().numpy().astype(bool)
        d = dev.cpu().view(torch.int16)
        h = host.view(torch.int16)
        assert mask.any()
        assert torch.equal(d[torch.from_numpy(mask)], h[torch.from_numpy(mask)])
        assert not d[torch.from_numpy(~mask)].any()
        eng.probs.fill_(0.5)
        eng.round()


def test_upload_rows_dma_runs_match_the_gather():
    """duchess_upload_rows (DMA per run of consecutive rows) over the survivor
    list read back to the host equals the gather over the device list, round
    after round; arbitrary order and duplicates in a caller's list are fine."""
    from paper_2509_24957_b200 import _lib
    from paper_2509_24957_b200.engine import BatchedDuchess
    knobs, traces, seeds = _setup(40, 8, 1.0)
    R, C = 6, 8
    eng = BatchedDuchess(traces, knobs, seeds, n_slots=R, pred_source=_lib.PRED_DEVICE,
                         queue=list(range(len(traces))), cycle=True)
    host = torch.randint(-1000, 1000, (R * C, 1, 3, 64), dtype=torch.int16).view(
        torch.bfloat16).pin_memory()
    eng.advance()
    for step in range(6):
        a = torch.zeros_like(host, device="cuda")
        b = torch.zeros_like(host, device="cuda")
        eng.upload_survivors(host, a)
        rows = eng.survivor_rows_host()
        assert len(rows) and sorted(rows) == sorted(np.nonzero(eng.t["row_mask"].cpu().numpy())[0])
        eng.upload_rows(host, b, rows[::-1].copy())
        torch.cuda.synchronize()
        assert torch.equal(a.view(torch.int16), b.view(torch.int16))
        eng.probs.fill_(0.5)
        eng.round()
    c = torch.zeros_like(host, device="cuda")
    eng.upload_rows(host, c, [5, 3, 4, 4, 40, 7])
    torch.cuda.synchronize()
    d, h = c.cpu().view(torch.int16), host.view(torch.int16)
    for r in range(R * C):
        listed = r in (3, 4, 5, 7, 40)
        assert torch.equal(d[r], h[r]) if listed else not d[r].any()
