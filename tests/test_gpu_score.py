"""K1 parity: fused pool + LayerNorm + linear probe vs the fp64 oracle on the
same (bf16-rounded) synthetic windows. Tolerance from north_star:
|logit_gpu - logit_ref| <= 1e-4 * max(|logit_ref|, 1)."""

import numpy as np
import pytest
import torch

from oracle import activations as oact
from oracle import port

pytestmark = pytest.mark.gpu


def _probe(H, L, seed):
    rng = np.random.default_rng(seed)
    w = rng.normal(0.0, 1.5 / np.sqrt(H), size=(L, H))
    g = rng.uniform(0.5, 1.5, size=(L, H))
    beta = rng.uniform(-0.1, 0.1, size=(L, H))
    b = rng.uniform(-0.2, 0.2, size=L)
    return w, b, g, beta


@pytest.mark.parametrize("dtype,T,H,L,rows,nsplit,threads", [
    (torch.float32, 1, 4096, 1, 64, 0, 0),          # C1 shape
    (torch.bfloat16, 32, 4096, 1, 48, 0, 0),        # C2 shape
    (torch.bfloat16, 32, 4096, 1, 16, 2, 256),      # split-merge path
    (torch.bfloat16, 32, 4096, 1, 16, 4, 128),
    (torch.bfloat16, 8, 5120, 4, 8, 0, 0),          # C3 shape (4 layers)
    (torch.float32, 3, 12, 1, 5, 0, 0),             # tiny, odd T
    (torch.bfloat16, 5, 10, 2, 4, 0, 0),            # unaligned -> generic kernel
    # T = 1: one warp per window (score_rows_kernel)
    (torch.bfloat16, 1, 5120, 4, 40, 0, 0),         # C3-T1 shape
    (torch.bfloat16, 1, 4096, 1, 300, 0, 0),
    (torch.bfloat16, 1, 4104, 2, 9, 0, 0),          # partial last vector column (nvec = 513)
    (torch.float32, 1, 1024, 3, 17, 0, 0),
    (torch.bfloat16, 1, 64, 1, 5000, 0, 0),         # tiny rows, > 1 unit per warp
])
def test_score_matches_oracle(dtype, T, H, L, rows, nsplit, threads):
    from paper_2509_24957_b200.probe import ProbeBank, Scorer, fill_windows
    w, b, g, beta = _probe(H, L, seed=H + L)
    bank = ProbeBank.from_linear(w, b, g, beta)
    acts = torch.empty((rows, L, T, H), dtype=dtype, device="cuda")
    req = torch.arange(rows, dtype=torch.int64, device="cuda") * 7 + 3
    tmpl = torch.arange(rows, dtype=torch.int32, device="cuda") % 5
    pos = torch.arange(rows, dtype=torch.int32, device="cuda") * 16 + 16
    fill_windows(acts, 1, req, tmpl, pos)
    scorer = Scorer(bank, rows * L, nsplit=nsplit, threads=threads)
    logit = torch.empty((rows, L), dtype=torch.float32, device="cuda")
    prob = torch.empty((rows, L), dtype=torch.float64, device="cuda")
    scorer(acts, logit, prob)
    torch.cuda.synchronize()
    bf16 = dtype == torch.bfloat16
    gpu_acts = acts.float().cpu().numpy()
    wgf = bank.wg.cpu().numpy().astype(np.float64)
    for r in range(rows):
        for l in range(L):
            win = oact.synth_window(1, int(req[r]), int(tmpl[r]), int(pos[r]), l, T, H, bf16)
            assert np.array_equal(win, gpu_acts[r, l]), "fill kernel != oracle regeneration"
            ref_logit, ref_prob = port.pooled_linear_probe(win, w[l], b[l], g[l], beta[l])
            got = float(logit[r, l])
            assert abs(got - ref_logit) <= 1e-4 * max(abs(ref_logit), 1.0), (r, l, got, ref_logit)
            # probability is sigmoid of the fp32 logit, computed in fp64
            p = 1.0 / (1.0 + np.exp(-np.float64(np.float32(got))))
            assert float(prob[r, l]) == pytest.approx(min(max(p, 1e-12), 1 - 1e-12), rel=1e-12)
    del wgf


@pytest.mark.parametrize("T", [4, 1])
def test_score_mask_skips_rows(T):
    from paper_2509_24957_b200.probe import ProbeBank, Scorer, fill_windows
    H, rows = 4096, 8
    w, b, g, beta = _probe(H, 1, seed=3)
    bank = ProbeBank.from_linear(w, b, g, beta)
    acts = torch.empty((rows, 1, T, H), dtype=torch.bfloat16, device="cuda")
    fill_windows(acts, 9)
    mask = torch.tensor([1, 0, 1, 0, 0, 1, 1, 0], dtype=torch.uint8, device="cuda")
    logit = torch.full((rows, 1), -7.0, device="cuda")
    prob = torch.full((rows, 1), -7.0, dtype=torch.float64, device="cuda")
    Scorer(bank, rows)(acts, logit, prob, row_mask=mask)
    torch.cuda.synchronize()
    for r in range(rows):
        if mask[r] == 0:
            assert float(logit[r, 0]) == -7.0 and float(prob[r, 0]) == -7.0
        else:
            assert float(prob[r, 0]) != -7.0


def test_score_deterministic():
    from paper_2509_24957_b200.probe import ProbeBank, Scorer, fill_windows
    H, T, rows = 4096, 32, 64
    w, b, g, beta = _probe(H, 1, seed=4)
    bank = ProbeBank.from_linear(w, b, g, beta)
    acts = torch.empty((rows, 1, T, H), dtype=torch.bfloat16, device="cuda")
    fill_windows(acts, 2)
    outs = []
    for ns in (2, 2):
        s = Scorer(bank, rows, nsplit=ns, threads=256)
        lg = torch.empty((rows, 1), device="cuda")
        pr = torch.empty((rows, 1), dtype=torch.float64, device="cuda")
        s(acts, lg, pr)
        outs.append(lg.clone())
    assert torch.equal(outs[0], outs[1])


def test_score_list_last_token_matches_oracle():
    """T = 1 through the survivor-list path (warp per window): only listed rows
    are written, in any list order, each within the north-star tolerance."""
    from paper_2509_24957_b200.probe import ProbeBank, Scorer, fill_windows
    rows, L, H = 700, 2, 5120
    w, b, g, beta = _probe(H, L, seed=11)
    bank = ProbeBank.from_linear(w, b, g, beta)
    acts = torch.empty((rows, L, 1, H), dtype=torch.bfloat16, device="cuda")
    req = torch.arange(rows, dtype=torch.int64, device="cuda") + 100
    tmpl = torch.zeros(rows, dtype=torch.int32, device="cuda")
    pos = torch.full((rows,), 32, dtype=torch.int32, device="cuda")
    fill_windows(acts, 4, req, tmpl, pos)
    pick = np.random.default_rng(2).permutation(rows)[:333]
    lst = torch.tensor(pick, dtype=torch.int32, device="cuda")
    cnt = torch.tensor([len(pick)], dtype=torch.int32, device="cuda")
    logit = torch.full((rows, L), 9.0, device="cuda")
    prob = torch.full((rows, L), 9.0, dtype=torch.float64, device="cuda")
    Scorer(bank, rows * L).score_list(acts, logit, prob, lst, cnt)
    torch.cuda.synchronize()
    lg = logit.cpu().numpy()
    chosen = set(int(r) for r in pick)
    for r in range(rows):
        if r not in chosen:
            assert (lg[r] == 9.0).all()
            continue
        if r % 7:
            continue
        for l in range(L):
            win = oact.synth_window(4, 100 + r, 0, 32, l, 1, H, True)
            ref, _ = port.pooled_linear_probe(win, w[l], b[l], g[l], beta[l])
            assert abs(float(lg[r, l]) - ref) <= 1e-4 * max(abs(ref), 1.0)
