"""tcgen05 MLP probe vs fp64 on the same bf16 operands (X and W1*ln_gain
rounded to bf16, fold constants from those values). Tolerance:
|logit - ref| <= 1e-4 * max(|ref|, 1) (fp32 accumulation)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _weights(K, NH, seed, bn=False):
    from paper_2509_24957_b200.predictor import MlpWeights
    rng = np.random.default_rng(seed)
    w1 = rng.normal(0, 1.0 / np.sqrt(K), (NH, K))
    w2 = rng.normal(0, 1.0 / np.sqrt(NH), (1, NH))
    return MlpWeights(K, [NH], 1, ["relu"], [w1, w2], [rng.normal(0, 0.1, NH), np.array([0.05])],
                      rng.uniform(0.5, 1.5, K), rng.uniform(-0.1, 0.1, K),
                      *([[rng.normal(0, 0.1, NH)], [rng.uniform(0.5, 2, NH)],
                         [rng.uniform(0.5, 1.5, NH)], [rng.normal(0, 0.1, NH)]] if bn
                        else [None] * 4))


def _ref(probe, X64):
    mu = X64.mean(axis=1, keepdims=True)
    sig = np.sqrt(((X64 - mu) ** 2).mean(axis=1, keepdims=True) + 1e-5)
    z = (X64 - mu) / sig
    h = np.maximum(z @ probe.W1g.T + probe.c[None, :], 0.0)
    return h @ probe.w2 + probe.b2


@pytest.mark.parametrize("M,K,NH,bn", [(300, 256, 512, False), (128, 64, 256, True),
                                       (1000, 5120, 2048, False), (257, 1024, 300, False)])
def test_tc_probe_matches_fp64(M, K, NH, bn):
    from paper_2509_24957_b200.mlp_probe import TensorCoreMlpProbe
    probe = TensorCoreMlpProbe(_weights(K, NH, M + K, bn))
    g = torch.Generator(device="cuda").manual_seed(M)
    X = (torch.randn((M, K), generator=g, device="cuda") * 1.3 + 0.2).to(torch.bfloat16)
    logit, prob = probe(X)
    torch.cuda.synchronize()
    ref = _ref(probe, X.float().cpu().numpy().astype(np.float64))
    got = logit.cpu().numpy().astype(np.float64)
    err = np.abs(got - ref) / np.maximum(np.abs(ref), 1.0)
    assert err.max() <= 1e-4, (err.max(), np.argmax(err))
    np.testing.assert_allclose(prob.cpu().numpy(), 1 / (1 + np.exp(-got.astype(np.float32).astype(np.float64))),
                               rtol=1e-12)


def test_tc_probe_matches_reference_mlp_forward_semantics():
    """Same network through the fp64 facade mlp_forward (predictor.py:126-151
    semantics): agreement up to the bf16 quantisation of X and W1."""
    from paper_2509_24957_b200.mlp_probe import TensorCoreMlpProbe
    from paper_2509_24957_b200.predictor import mlp_forward_batch
    w = _weights(512, 256, 3)
    probe = TensorCoreMlpProbe(w)
    X = torch.randn((64, 512), device="cuda").to(torch.bfloat16)
    logit, _ = probe(X)
    ref, _ = mlp_forward_batch(w, X.float().cpu().numpy())
    assert np.abs(logit.cpu().numpy() - ref[:, 0]).max() < 0.05
