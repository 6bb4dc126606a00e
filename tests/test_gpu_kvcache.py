"""K3 in the round (duchess_kv_round) vs the paged-KV restatement
(oracle/kvcache.py) replaying the oracle's DuchessRun (GPU, through the
C-ABI): after the first advance and after every duchess_round, every
occupied slot's arena — block-table rows in local block ids, refcounts, free
stack, high-water mark — equals the oracle arena of the request it serves at
the same round; the forks' tail copies move the root's partial block bytes."""

import random

import numpy as np
import pytest
import torch

from oracle import kvcache, port
from tests.golden_util import case_knobs, case_traces, load

pytestmark = pytest.mark.gpu


def _gen(n_req, templates, c, preset, seed=7):
    if preset == "gsm8k":
        knobs = port.Knobs(max_branches=c, interval_tokens=16, early_term_threshold=0.70,
                           early_term_rounds=2, branch_out_temperature=1.0,
                           consensus_frac=0.6, coverage_frac=0.8)
        params = port.GenParams(level_median_tokens=(180, 220, 260, 300, 350),
                                level_correct_prob=(0.92, 0.88, 0.84, 0.80, 0.75),
                                templates_per_request=templates, probe_stride=16)
    else:
        knobs = port.Knobs(max_branches=c, interval_tokens=80, early_term_threshold=0.80,
                           early_term_rounds=2, branch_out_temperature=0.8,
                           consensus_frac=0.6, coverage_frac=0.8)
        params = port.GenParams(level_median_tokens=(340, 460, 640, 840, 1180),
                                level_correct_prob=(0.85, 0.78, 0.70, 0.62, 0.52),
                                distractor_count=10, probe_stride=40,
                                templates_per_request=templates)
    traces = port.generate(params, n_req, seed=seed)
    master = random.Random(11)
    return knobs, traces, [master.getrandbits(64) for _ in traces]


def _run(traces, knobs, seeds, rho, slots, P, kv_bytes=64, block_tokens=16, check_bytes=True):
    from paper_2509_24957_b200 import _lib
    from paper_2509_24957_b200.engine import BatchedDuchess
    from paper_2509_24957_b200.kvfork import PagedKVCache
    eng = BatchedDuchess(traces, knobs, seeds, n_slots=slots, pred_source=_lib.PRED_TRACE,
                         rho=rho)
    kv = PagedKVCache(eng, blocks_per_slot=P, kv_bytes_per_token=kv_bytes,
                      block_tokens=block_tokens)
    g = torch.Generator(device="cuda").manual_seed(3)
    if kv_bytes:
        kv.t["kv_pool"].copy_(torch.randint(0, 256, kv.t["kv_pool"].shape, generator=g,
                                            device="cuda", dtype=torch.int32).to(torch.uint8))
    oracle = [kvcache.replay(port.DuchessRequest(t, knobs, random.Random(s), rho=rho), P,
                             block_tokens) for t, s in zip(traces, seeds)]
    seen = set()
    n_jobs = 0

    def check():
        nonlocal n_jobs
        rounds = eng.t["rounds"].cpu().numpy()
        for r in range(eng.R):
            snap = kv.slot_snapshot(r)
            p = snap.pop("owner")
            snap.pop("peak")
            if p < 0:
                assert snap["rows"] == {} and snap["hwm"] == 0, f"idle slot {r}"
                continue
            i = int(rounds[r]) - 1           # rounds counts the round in flight (phase 1)
            assert snap == oracle[p][i], f"slot {r} request {p} after round {i}"
            seen.add((p, i))
        if check_bytes and kv_bytes:
            jc = kv.t["job_count"].cpu().numpy()
            jobs = kv.t["jobs"].view(eng.R, eng.C, 4).cpu().numpy()
            pool = kv.t["kv_pool"].view(-1, block_tokens * kv_bytes)
            for r in range(eng.R):
                for q in range(int(jc[r])):
                    src, dst, tok = (int(x) for x in jobs[r, q, :3])
                    n = tok * kv_bytes
                    assert torch.equal(pool[src, :n], pool[dst, :n]), "tail copy"
                    n_jobs += 1

    eng.advance()
    kv.round()
    check()
    for _ in range(100000):
        eng.round()
        kv.round()
        check()
        if eng.all_done():
            break
    cnt = kv.counters()
    assert cnt["overflow"] == 0
    # every request's every oracle call was compared
    assert seen == {(p, i) for p in range(len(traces)) for i in range(len(oracle[p]) - 1)}
    return cnt, n_jobs


@pytest.mark.parametrize("case", load("decisions.json")[:6], ids=lambda c: c["name"])
def test_kv_round_matches_oracle_golden_workloads(case):
    traces = case_traces(case)
    seeds = [int(r["seed"]) for r in case["requests"]]
    _run(traces, case_knobs(case), seeds, case["rho"], slots=min(5, len(traces)), P=512)


@pytest.mark.parametrize("preset,c,bt", [("gsm8k", 8, 16), ("math", 16, 16), ("math", 16, 32),
                                         ("gsm8k", 8, 24)])
def test_kv_round_matches_oracle_forks_heavy(preset, c, bt):
    """Survivors sit on multiples of interval_tokens (a partial chunk ends the
    branch), so most forks need a tail copy only when the block size does not
    divide the interval (math-like i = 80 with 32-token blocks, gsm8k-like
    i = 16 with 24-token blocks); otherwise only a child forked from a
    same-round child clamped to its natural length (orchestrator.py:263)
    starts off a block boundary."""
    knobs, traces, seeds = _gen(24, 64, c, preset)
    cnt, n_jobs = _run(traces, knobs, seeds, 0.7, slots=6, P=c * 4096 // bt, block_tokens=bt)
    assert cnt["blocks_allocated"] > 0 and cnt["blocks_released"] > 0
    if knobs.interval_tokens % bt:
        assert n_jobs > 20 and cnt["tail_bytes"] > 0


@pytest.mark.parametrize("mode", ["lead", "overlap"])
def test_serving_loop_kv_overlapped_matches_oracle(mode):
    """The measured loop with K3 (bench.py default C2 with the KV cache, scaled down): two
    request shards, K1 + round + K3 per shard stream — K3 launched right after
    its round with the next scorer streaming beside it ("lead", the default),
    or beside the next round's scorer ("overlap"). After every K3 (taken
    right before the next round) each occupied slot's arena equals the
    oracle arena of its request, replayed from the oracle DuchessRun fed the
    device's probabilities (predictor=, orchestrator.py:319-327)."""
    import bench
    from paper_2509_24957_b200.probe import ProbeBank
    from paper_2509_24957_b200.scheduler import difficulty_queue
    from paper_2509_24957_b200.serving import ShardedEngine, keyed_fill
    T, H, L, R, pool, seed, P = 4, 512, 1, 32, 96, 5, 1024
    cfg = dict(bench.CONFIGS["c2"], R=R, pool=pool, T=T, H=H, L=L)
    traces, knobs, seeds = bench.make_workload(cfg, seed=1000)
    w, b, g, beta = bench.make_probe(H, L)
    bank = ProbeBank.from_linear(w, b, g, beta)
    queue = difficulty_queue([t.difficulty for t in traces])
    # lead: K3 right after each round, the next scorer streaming beside it
    # (DUCHESS_SCORE_NO_INPUT_WAIT); overlap: K3 beside the next round's scorer
    srv = ShardedEngine(traces, knobs, seeds, bank, n_slots=R, shards=2, queue=queue,
                        cycle=False, T=T, dtype=torch.bfloat16,
                        kv=dict(block_tokens=16, blocks_per_slot=P, kv_bytes_per_token=64),
                        kv_mode=mode)
    keyed = keyed_fill(seed)
    snaps = [[] for _ in range(2)]
    preds = [[] for _ in range(2)]
    pending = [None, None]

    def fill(k, eng, acts):                      # the round in flight: its survivors
        keyed(k, eng, acts)
        pending[k] = [eng.t[n].clone() for n in ("row_mask", "row_req", "row_tmpl", "row_pos")]

    def before(k, eng):
        snaps[k].append((srv.shards[k]["kv"].state_copy(), eng.t["rounds"].clone()))

    def after(k, eng):
        preds[k].append(pending[k] + [eng.t["step_pred"].clone()])

    srv.run(max_rounds=2000, fill=fill, after_round=after, before_round=before)
    torch.cuda.synchronize()
    seen = {}
    for k in range(2):
        for mask, req, tm, pos, pred in preds[k]:
            mask = mask.cpu().numpy().astype(bool)
            req, tm, pos, pred = (x.cpu().numpy() for x in (req, tm, pos, pred))
            for row in np.nonzero(mask)[0]:
                seen[(int(req[row]), int(tm[row]), int(pos[row]))] = float(pred[row])
    oracle = []
    for p, trace in enumerate(traces):
        index = {id(tp): j for j, tp in enumerate(trace.templates)}

        def predictor(tmpl, position, _rng, p=p, index=index):
            return seen[(p, index[id(tmpl)], position)]

        req = port.DuchessRequest(trace, knobs, random.Random(seeds[p]), predictor=predictor)
        oracle.append(kvcache.replay(req, P))
    checked = set()
    for k in range(2):
        kv = srv.shards[k]["kv"]
        for state, rounds in snaps[k]:
            rounds = rounds.cpu().numpy()
            for r in range(kv.R):
                snap = kv.slot_snapshot(r, state)
                p = snap.pop("owner")
                snap.pop("peak")
                if p < 0:
                    continue
                i = int(rounds[r]) - 1
                assert snap == oracle[p][i], f"shard {k} slot {r} request {p} after round {i}"
                checked.add((p, i))
    assert len(checked) > 500
    assert srv.kv_counters()["overflow"] == 0
