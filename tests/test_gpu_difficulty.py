"""Tensor-core difficulty classifier: tcgen05 hidden layers
with LayerNorm / batch-norm / GeLU fused, checked against the fp64 forward
(the facade's duchess_mlp_forward and the CPU oracle restatement of
predictor.py:126-151). Levels (argmax + 1) must equal the fp64 ones for every
row; logits within the bf16-chain tolerance stated below."""

import numpy as np
import pytest
import torch

from oracle import port

pytestmark = pytest.mark.gpu


def complexity_mlp(seed, dims, head=5, act="gelu", batchnorm=True, layernorm=True):
    from paper_2509_24957_b200.predictor import MlpWeights
    rng = np.random.default_rng(seed)
    hid = list(dims[1:])
    full = [dims[0], *hid, head]
    W = [rng.normal(0, 1 / np.sqrt(full[k]), (full[k + 1], full[k])) for k in range(len(full) - 1)]
    W[-1] *= 3.0                                    # spread the 5 logits
    b = [rng.normal(0, 0.1, full[k + 1]) for k in range(len(full) - 1)]
    bn = dict(bn_mean=[rng.normal(0, 0.1, d) for d in hid],
              bn_var=[rng.uniform(0.5, 2.0, d) for d in hid],
              bn_gain=[rng.uniform(0.5, 1.5, d) for d in hid],
              bn_bias=[rng.uniform(-0.1, 0.1, d) for d in hid]) if batchnorm else {}
    ln = dict(ln_gain=rng.uniform(0.5, 1.5, dims[0]),
              ln_bias=rng.uniform(-0.1, 0.1, dims[0])) if layernorm else {}
    return MlpWeights(dims[0], hid, head, [act] * len(hid), W, b, **ln, **bn)


def activations(seed, M, H):
    rng = np.random.default_rng(seed)
    x = rng.normal(0, 1, (M, H))
    x[:, 257::512] *= 20.0                          # outlier channels, as in real activations
    return x


@pytest.mark.parametrize("dims,act,bn,ln,M", [
    ((4096, 2048, 1024, 512), "gelu", True, True, 1000),    # the paper's complexity MLP
    ((512, 256, 256), "relu", False, True, 37),
    ((1024, 512), "gelu", True, False, 300),
])
def test_tc_classifier_matches_fp64(dims, act, bn, ln, M):
    from paper_2509_24957_b200.difficulty import TensorCoreClassifier
    from paper_2509_24957_b200.predictor import mlp_forward_batch
    w = complexity_mlp(1, dims, act=act, batchnorm=bn, layernorm=ln)
    X = activations(2, M, dims[0])
    clf = TensorCoreClassifier(w)
    lg = clf.logits(X).cpu().numpy()
    ref_logits, ref_probs = mlp_forward_batch(w, X)
    err = np.abs(lg - ref_logits).max()
    # bf16 operands and bf16 inter-layer activations, fp32 accumulation: the
    # logit error stays far below the fallback margin / 2 (0.125)
    assert err < 0.05, err
    levels = clf.predict_levels(X)
    assert (levels == ref_probs.argmax(axis=1) + 1).all()
    for i in range(3):                              # fp64 device path == CPU oracle
        o_logits, _ = port.mlp_forward(w, X[i])
        assert np.allclose(ref_logits[i], o_logits, rtol=1e-9, atol=1e-9)


@pytest.mark.parametrize("offset,scale", [(1000.0, 1.0), (-3.0e4, 0.01), (5.0, 100.0)])
def test_tc_classifier_large_common_offset(offset, scale):
    """Rows with a large common offset / odd scale: the input is
    LayerNorm-normalised in fp64 before the bf16 cast, so the tensor-core
    logits stay within the calibrated margin's half and the levels equal the
    fp64 forward's."""
    from paper_2509_24957_b200.difficulty import TensorCoreClassifier
    from paper_2509_24957_b200.predictor import mlp_forward_batch
    w = complexity_mlp(3, (1024, 512, 256), act="gelu", batchnorm=True, layernorm=True)
    X = activations(4, 400, 1024) * scale + offset
    clf = TensorCoreClassifier(w)
    lg = clf.logits(X).cpu().numpy()
    ref_logits, ref_probs = mlp_forward_batch(w, X)
    assert np.abs(lg - ref_logits).max() < clf.margin / 2, (np.abs(lg - ref_logits).max(),
                                                            clf.margin)
    assert (clf.predict_levels(X) == ref_probs.argmax(axis=1) + 1).all()


def test_tc_classifier_shape_errors():
    from paper_2509_24957_b200.difficulty import TensorCoreClassifier
    from paper_2509_24957_b200.predictor import WeightFormatError
    w = complexity_mlp(3, (512, 256))
    clf = TensorCoreClassifier(w)
    with pytest.raises(WeightFormatError):
        clf.logits(np.zeros((4, 500)))
    with pytest.raises(ValueError):
        TensorCoreClassifier(complexity_mlp(3, (500, 256)))


def test_predict_difficulty_batch_equals_single_calls():
    from paper_2509_24957_b200.predictor import predict_difficulty, predict_difficulty_batch
    w = complexity_mlp(4, (512, 256, 256))
    X = activations(5, 40, 512)
    batch = predict_difficulty_batch(w, X)
    single = [predict_difficulty("mlp", activation=x, weights=w) for x in X[:10]]
    assert batch[:10] == single
    assert set(batch) <= {1, 2, 3, 4, 5}


@pytest.mark.parametrize("dtype,K", [(torch.bfloat16, 4096), (torch.bfloat16, 1032),
                                     (torch.bfloat16, 512), (torch.bfloat16, 8192),
                                     (torch.float32, 4096), (torch.float32, 200),
                                     (torch.float64, 512)])
def test_row_normalize_matches_fp64(dtype, K):
    """duchess_row_normalize (the classifier's input LayerNorm pass,
    predictor.py:134-136) on bf16 / fp32 / fp64 rows: z = (x - mean) / std
    with fp64 statistics, stored bf16 — equal to the fp64 formula rounded to
    bf16 up to one bf16 ulp (the fp64 sums' order differs)."""
    from paper_2509_24957_b200 import _lib
    lib = _lib.load()
    g = torch.Generator(device="cuda").manual_seed(K)
    x = (torch.randn((300, K), generator=g, device="cuda", dtype=torch.float64) * 3 + 50).to(dtype)
    z = torch.empty((300, K), dtype=torch.bfloat16, device="cuda")
    dt = {torch.bfloat16: _lib.BF16, torch.float32: _lib.F32, torch.float64: _lib.F64}[dtype]
    _lib.check(lib.duchess_row_normalize(x.data_ptr(), dt, 300, K, z.data_ptr(),
                                         _lib.stream_handle()), "row_normalize")
    xd = x.double()
    ref = (xd - xd.mean(1, keepdim=True)) / torch.sqrt(xd.var(1, unbiased=False, keepdim=True) + 1e-5)
    got = z.double()
    ulp = ref.abs().clamp_min(2 ** -126) * 2 ** -7
    assert bool(((got - ref).abs() <= ulp).all())


@pytest.mark.parametrize("K,n_out,M", [(512, 5, 3001), (256, 5, 17), (200, 5, 40), (1024, 5, 999),
                                       (512, 3, 500)])
def test_head_logits_match_fp64(K, n_out, M):
    """duchess_head_logits (the classifier's output layer over the last hidden
    bf16 vectors): the register-weight kernel (5 outputs, K <= 512), the
    vector kernel and the scalar fallback all equal the fp64 dot of the same
    bf16 inputs within fp32 accumulation error."""
    from paper_2509_24957_b200 import _lib
    lib = _lib.load()
    g = torch.Generator(device="cuda").manual_seed(K * 7 + n_out)
    h = torch.randn((M, K), generator=g, device="cuda").to(torch.bfloat16)
    W = torch.randn((n_out, K), generator=g, device="cuda") / np.sqrt(K)
    b = torch.randn(n_out, generator=g, device="cuda")
    out = torch.empty((M, n_out), device="cuda")
    _lib.check(lib.duchess_head_logits(h.data_ptr(), M, K, W.data_ptr(), b.data_ptr(), n_out,
                                       out.data_ptr(), _lib.stream_handle()), "head_logits")
    ref = h.double() @ W.double().T + b.double()
    np.testing.assert_allclose(out.double().cpu().numpy(), ref.cpu().numpy(), rtol=1e-5, atol=1e-5)
