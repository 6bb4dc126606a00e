"""Extended randomised parity sweep (seeds 40..439 of tests/test_gpu_random_configs.py, both
round-kernel modes); run under gpurun. Prints the failing (seed, mode) pairs."""
import sys, traceback
sys.path.insert(0, ".")
from tests.test_gpu_random_configs import test_random_config_matches_oracle as t
bad = []
for seed in range(40, 440):
    for mode in ("split", "round"):
        try:
            t(seed, mode)
        except Exception as e:
            bad.append((seed, mode, repr(e)[:200]))
print("failures:", len(bad))
for b in bad[:10]:
    print(b)
