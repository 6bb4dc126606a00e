"""Body of __graft_entry__.smoke(): one short run of the serving loop
(serving.ShardedEngine: two request shards on two CUDA streams, each round
K1 duchess_score_active_ex + K2 duchess_round + K3 duchess_kv_round on a paged
KV cache) on cuda:0, checked against the CPU oracle (oracle/ is the checker
only): logits and every RoundReport; the KV cache must not overflow."""

from __future__ import annotations

import random

import numpy as np


def run_smoke() -> None:
    import torch

    from oracle import activations as oact
    from oracle import port
    from paper_2509_24957_b200 import _lib
    from paper_2509_24957_b200.engine import decode_round
    from paper_2509_24957_b200.probe import ProbeBank
    from paper_2509_24957_b200.serving import ShardedEngine, keyed_fill

    assert torch.cuda.is_available(), "smoke() needs cuda:0"
    H, T, L, R, seed = 1024, 4, 1, 4, 3
    knobs = port.Knobs(max_branches=4, interval_tokens=16, early_term_threshold=0.6,
                       early_term_rounds=1, branch_out_temperature=0.8)
    traces = port.generate(port.GenParams(level_median_tokens=(60, 70, 80, 90, 100),
                                          templates_per_request=8), 6, seed=5)
    seeds = [random.Random(9).getrandbits(64) + i for i in range(len(traces))]
    rng = np.random.default_rng(1)
    w = rng.normal(0, 1.5 / np.sqrt(H), size=(1, H))
    bank = ProbeBank.from_linear(w, [0.05])
    P = 256                                          # KV blocks per slot arena
    srv = ShardedEngine(traces, knobs, seeds, bank, n_slots=R, shards=2, T=T,
                        dtype=torch.bfloat16,
                        kv=dict(block_tokens=16, blocks_per_slot=P, kv_bytes_per_token=64))
    C = knobs.max_branches
    fill = keyed_fill(seed)
    seen, reports = {}, {}

    def check_round(k, eng):
        torch.cuda.current_stream().synchronize()
        t = eng.t
        mask = t["row_mask"].cpu().numpy().astype(bool)
        req, tm, pos = (t[n].cpu().numpy() for n in ("row_req", "row_tmpl", "row_pos"))
        pending[k] = (mask, req, tm, pos)

    pending = [None, None]

    def fill_and_record(k, eng, acts):
        fill(k, eng, acts)
        check_round(k, eng)

    def after(k, eng):
        torch.cuda.current_stream().synchronize()
        mask, req, tm, pos = pending[k]
        pr = eng.t["step_pred"].cpu().numpy()
        lg = srv.shards[k]["logit"].cpu().numpy()[:, 0]
        for row in np.nonzero(mask)[0]:
            key = (int(req[row]), int(tm[row]), int(pos[row]))
            seen[key] = float(pr[row])
            win = oact.synth_window(seed, *key, 0, T, H, True)
            ref, _ = port.pooled_linear_probe(win, w[0], 0.05, None, None)
            assert abs(float(lg[row]) - ref) <= 1e-4 * max(abs(ref), 1.0), (key, lg[row], ref)
        for p, rep in decode_round(eng.t["round_rec"].cpu().numpy(),
                                   eng.t["actions"].cpu().numpy(), srv.Rs, C):
            reports.setdefault(p, []).append(rep)

    srv.run(max_rounds=1000, fill=fill_and_record, after_round=after)
    assert int(srv.counters()[_lib.CNT_AMBIGUOUS]) == 0
    assert srv.kv_counters()["overflow"] == 0 and srv.kv_counters()["blocks_allocated"] > 0
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
