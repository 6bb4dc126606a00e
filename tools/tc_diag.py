"""Diagnostics for the tcgen05 MLP probe: max / median relative logit error vs
the fp64 reference over a sweep of (M, K, NH) shapes and input means (run under
gpurun)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from tests.test_gpu_mlp_tc import _weights, _ref  # noqa: E402
from paper_2509_24957_b200.mlp_probe import TensorCoreMlpProbe  # noqa: E402

for M, K, NH in [(128, 64, 256), (128, 256, 256), (128, 1024, 256), (128, 2048, 256), (128, 5120, 256),
                 (128, 256, 512), (128, 256, 1024), (128, 256, 2048), (1000, 256, 256), (128, 512, 768)]:
    probe = TensorCoreMlpProbe(_weights(K, NH, 7))
    g = torch.Generator(device="cuda").manual_seed(1)
    for mean in (0.0, 0.2):
        X = (torch.randn((M, K), generator=g, device="cuda") * 1.3 + mean).to(torch.bfloat16)
        logit, _ = probe(X)
        torch.cuda.synchronize()
        ref = _ref(probe, X.float().cpu().numpy().astype(np.float64))
        got = logit.cpu().numpy().astype(np.float64)
        err = np.abs(got - ref) / np.maximum(np.abs(ref), 1.0)
        print(f"M={M} K={K} NH={NH} mean={mean}: max_err={err.max():.2e} med={np.median(err):.2e} "
              f"|ref|~{np.abs(ref).mean():.2f}")
