"""Body of __graft_entry__.smoke(): one short end-to-end run of the hot path
(advance -> fill -> K1 score -> decide) on cuda:0, checked against the CPU
oracle (oracle/ is the checker only)."""

from __future__ import annotations

import random

import numpy as np


def run_smoke() -> None:
    import torch

    from oracle import activations as oact
    from oracle import port
    from paper_2509_24957_b200 import _lib
    from paper_2509_24957_b200.engine import BatchedDuchess
    from paper_2509_24957_b200.probe import ProbeBank, Scorer, fill_windows

    assert torch.cuda.is_available(), "smoke() needs cuda:0"
    H, T, L, R, seed = 1024, 4, 1, 2, 3
    knobs = port.Knobs(max_branches=4, interval_tokens=16, early_term_threshold=0.6,
                       early_term_rounds=1, branch_out_temperature=0.8)
    traces = port.generate(port.GenParams(level_median_tokens=(60, 70, 80, 90, 100),
                                          templates_per_request=8), 3, seed=5)
    seeds = [random.Random(9).getrandbits(64) + i for i in range(len(traces))]
    rng = np.random.default_rng(1)
    w = rng.normal(0, 1.5 / np.sqrt(H), size=(1, H))
    bank = ProbeBank.from_linear(w, [0.05])
    eng = BatchedDuchess(traces, knobs, seeds, n_slots=R, pred_source=_lib.PRED_DEVICE)
    C = knobs.max_branches
    acts = torch.zeros((R * C, L, T, H), dtype=torch.bfloat16, device="cuda")
    scorer = Scorer(bank, R * C)
    logit = torch.zeros((R * C, L), device="cuda")
    seen = {}

    def score(e):
        t = e.t
        fill_windows(acts, seed, t["row_req"], t["row_tmpl"], t["row_pos"], t["row_mask"])
        scorer(acts, logit, e.probs.view(R * C, L), row_mask=t["row_mask"])

    reports = {}
    for _ in range(1000):
        eng.step(score_fn=score)
        t = eng.t
        mask = t["row_mask"].cpu().numpy().astype(bool)
        req, tm, pos = (t[k].cpu().numpy() for k in ("row_req", "row_tmpl", "row_pos"))
        pr, lg = eng.probs.cpu().numpy(), logit.cpu().numpy()[:, 0]
        for row in np.nonzero(mask)[0]:
            key = (int(req[row]), int(tm[row]), int(pos[row]))
            seen[key] = float(pr[row])
            win = oact.synth_window(seed, *key, 0, T, H, True)
            ref, _ = port.pooled_linear_probe(win, w[0], 0.05, None, None)
            assert abs(float(lg[row]) - ref) <= 1e-4 * max(abs(ref), 1.0), (key, lg[row], ref)
        for p, rep in eng.round_reports():
            reports.setdefault(p, []).append(rep)
        if eng.all_done():
            break
    for p, trace in enumerate(traces):
        index = {id(x): j for j, x in enumerate(trace.templates)}
        req_o = port.DuchessRequest(trace, knobs, random.Random(seeds[p]),
                                    predictor=lambda tm_, ps, _r, p=p, ix=index:
                                    seen[(p, ix[id(tm_)], ps)])
        want = []
        while not req_o.done:
            r = req_o.step()
            want.append((r.round_index, r.decoding_branches, r.max_chunk, r.decode_tokens,
                         r.probes, [tuple(a) for a in r.actions], r.done))
        assert reports[p] == want, f"smoke: request {p} diverged from the oracle"
