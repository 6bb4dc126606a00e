"""The paper's probe (LN -> 2048 ReLU -> 1024 ReLU -> 1) for L
probe layers on the tensor cores (MlpProbeBank: duchess_tc_linear_grouped +
duchess_mlp_probe_tc_grouped) vs fp64.

Tolerances, written here: against fp64 on the SAME bf16 operands (X as read,
W1 * ln_gain and W2 rounded to bf16, h1 rounded to bf16 where the device
stores it) the only differences are fp32 accumulation and the rounding of h1
near bf16 ties, |logit - ref| <= 2e-3 * max(|ref|, 1); against the
reference's fp64 mlp_forward on the bf16 inputs (predictor.py:126-151,
unrounded weights), the bf16 weight / hidden quantisation bound
|logit - ref| <= 0.05 * max(|ref|, 1)."""

import numpy as np
import pytest
import torch

from oracle import port

pytestmark = pytest.mark.gpu


def _bf16(x):
    from paper_2509_24957_b200.hostmath import bf16_round_np
    return bf16_round_np(x)


def same_operand_ref(bank, X64):
    M = X64.shape[0]
    out = np.zeros((M, bank.G))
    h = bank.host
    for l in range(bank.G):
        x = X64[:, l, :]
        mu = x.mean(axis=1, keepdims=True)
        sig = np.sqrt(((x - mu) ** 2).mean(axis=1, keepdims=True) + 1e-5)
        a = np.maximum(((x - mu) / sig) @ h["W1"][l].T + h["C1"][l], 0.0)
        if len(bank.hidden) == 2:
            a = np.maximum(_bf16(a) @ h["W2"][l].T + h["c2"][l], 0.0)
        out[:, l] = a @ h["w3"][l] + h["b3"][l]
    return out


@pytest.mark.parametrize("M,G,K,hidden", [(300, 4, 512, (512, 256)), (1000, 4, 5120, (2048, 1024)),
                                          (257, 2, 1024, (256, 256)), (129, 3, 768, (512,))])
def test_paper_probe_matches_fp64(M, G, K, hidden):
    from paper_2509_24957_b200.mlp_probe import MlpProbeBank
    probes = MlpProbeBank.paper_probes(G, K, seed=M, hidden=hidden)
    bank = MlpProbeBank(probes)
    g = torch.Generator(device="cuda").manual_seed(M)
    X = (torch.randn((M, G, K), generator=g, device="cuda") * 1.3 + 0.2).to(torch.bfloat16)
    logit = torch.empty((M, G), device="cuda")
    prob = torch.empty((M, G), dtype=torch.float64, device="cuda")
    bank(X, logit, prob)
    torch.cuda.synchronize()
    X64 = X.float().cpu().numpy().astype(np.float64)
    got = logit.cpu().numpy().astype(np.float64)
    ref = same_operand_ref(bank, X64)
    err = np.abs(got - ref) / np.maximum(np.abs(ref), 1.0)
    print("same-operand max rel err", err.max(), "logit range", ref.min(), ref.max())
    assert err.max() <= 2e-3, (err.max(), np.unravel_index(np.argmax(err), err.shape))
    full = np.stack([np.array([port.mlp_forward(probes[l], X64[i, l])[0][0]
                               for i in range(min(M, 64))]) for l in range(G)], axis=1)
    err2 = np.abs(got[:full.shape[0]] - full) / np.maximum(np.abs(full), 1.0)
    print("vs fp64 mlp_forward max rel err", err2.max())
    assert err2.max() <= 0.05
    np.testing.assert_allclose(prob.cpu().numpy(),
                               np.clip(1 / (1 + np.exp(-got)), 1e-12, 1 - 1e-12), rtol=1e-6)


def test_paper_probe_drives_decisions_in_serving_loop():
    """The serving loop (serving.ShardedEngine, two request shards) scoring
    with the paper's MLP probe (L = 2 layers, T = 1 last-token windows keyed by
    (request, template, position)): every request's RoundReports and outcome
    equal the oracle DuchessRun fed the device probabilities through
    predictor= (orchestrator.py:319-327, :358-363), the probability is the mean
    over layers of the per-layer probe, and sampled logits match fp64 on the
    same bf16 operands (tolerance above)."""
    import random

    import bench
    from oracle import activations as oact
    from paper_2509_24957_b200.engine import decode_round
    from paper_2509_24957_b200.mlp_probe import MlpProbeBank
    from paper_2509_24957_b200.scheduler import difficulty_queue
    from paper_2509_24957_b200.serving import ShardedEngine, keyed_fill
    from tests.golden_util import port_report_tuple
    L, H, R, pool, seed = 2, 512, 32, 96, 9
    cfg = dict(bench.CONFIGS["c3t1"], R=R, pool=pool, H=H, L=L, c=16)
    traces, knobs, seeds = bench.make_workload(cfg, seed=1000)
    probes = MlpProbeBank.paper_probes(L, H, seed=4, hidden=(512, 256))
    bank = MlpProbeBank(probes)
    queue = difficulty_queue([t.difficulty for t in traces])
    srv = ShardedEngine(traces, knobs, seeds, bank, n_slots=R, shards=2, queue=queue,
                        cycle=False, T=1, dtype=torch.bfloat16)
    keyed = keyed_fill(seed)
    snaps, pending = [[], []], [None, None]

    def fill(k, eng, acts):
        keyed(k, eng, acts)
        pending[k] = [eng.t[n].clone() for n in ("row_mask", "row_req", "row_tmpl", "row_pos")]

    def after(k, eng):
        snaps[k].append(pending[k] + [eng.t["step_pred"].clone(), srv.shards[k]["logit"].clone(),
                                      eng.t["round_rec"].clone(), eng.t["actions"].clone()])

    srv.run(max_rounds=2000, fill=fill, after_round=after)
    torch.cuda.synchronize()
    seen, logits, reports = {}, {}, {}
    for k in range(2):
        for mask, req, tm, pos, pred, lg, rec, act in snaps[k]:
            mask = mask.cpu().numpy().astype(bool)
            req, tm, pos, pred, lg = (x.cpu().numpy() for x in (req, tm, pos, pred, lg))
            for row in np.nonzero(mask)[0]:
                key = (int(req[row]), int(tm[row]), int(pos[row]))
                seen[key] = float(pred[row])
                logits[key] = lg[row].copy()
            for p, rep in decode_round(rec.cpu().numpy(), act.cpu().numpy(), srv.Rs,
                                       knobs.max_branches):
                reports.setdefault(p, []).append(rep)
    rng = random.Random(0)
    keys = rng.sample(sorted(seen), 96)
    X64 = np.stack([np.stack([oact.synth_window(seed, *key, l, 1, H, True)[0] for l in range(L)])
                    for key in keys])
    ref = same_operand_ref(bank, X64)
    for i, key in enumerate(keys):
        got = logits[key]
        assert np.all(np.abs(got - ref[i]) <= 2e-3 * np.maximum(np.abs(ref[i]), 1.0)), key
        pm = np.mean(np.clip(1 / (1 + np.exp(-got.astype(np.float64))), 1e-12, 1 - 1e-12))
        assert abs(seen[key] - pm) <= 1e-6, key
    outcomes = srv.outcomes()
    assert sorted(outcomes) == list(range(len(traces)))
    for p, trace in enumerate(traces):
        index = {id(tp): j for j, tp in enumerate(trace.templates)}

        def predictor(tmpl, position, _rng, p=p, index=index):
            return seen[(p, index[id(tmpl)], position)]

        req = port.DuchessRequest(trace, knobs, random.Random(seeds[p]), predictor=predictor)
        want = []
        while not req.done:
            want.append(port_report_tuple(req.step()))
        assert reports[p] == want, f"request {p}"
        assert outcomes[p]["final"] == req.outcome.final
