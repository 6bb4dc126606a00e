"""cProfile of one run_simulation call (4096 requests) on the GPU box."""
import cProfile
import pstats
import sys
sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2509_24957_b200.orchestrator import OrchestratorConfig  # noqa: E402
from paper_2509_24957_b200.predictor import SyntheticPredictorConfig  # noqa: E402
from paper_2509_24957_b200.scheduler import ArrivalConfig, gen_arrivals  # noqa: E402
from paper_2509_24957_b200.simengine import TimingModel, run_simulation  # noqa: E402
from paper_2509_24957_b200.workload import SyntheticParams, generate_synthetic  # noqa: E402

n = 4096
wl = generate_synthetic(SyntheticParams(**bench.PRESET_GEN["math-like"]), n, seed=21)
arr = gen_arrivals(ArrivalConfig(rate_qpm=30.0, n_requests=n, seed=3))
orch = OrchestratorConfig(max_branches=10, **bench.PRESET_KNOBS["math-like"])
kw = dict(synthetic=SyntheticPredictorConfig(rho=0.8), difficulty_mode="noisy-label")
run_simulation(wl, orch, "duchess", "easiest-predicted", arr, TimingModel(), 9, **kw)
pr = cProfile.Profile()
pr.enable()
run_simulation(wl, orch, "duchess", "easiest-predicted", arr, TimingModel(), 9, **kw)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(22)
