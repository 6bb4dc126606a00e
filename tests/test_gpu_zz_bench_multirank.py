"""bench.py's N > 1 path (torchrun, one process per rank, barrier + max-over-ranks
timing, rank 0 prints one JSON line) run with two ranks on the box's GPU(s).
The collectives go over gloo (DUCHESS_BENCH_BACKEND, test only) so two ranks
can share one GPU; on an 8-GPU node the same code runs with NCCL."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("config,extra", [("c3", ["--slots", "64"]), ("c2", ["--slots", "64"]),
                                          ("c5", [])])
def test_bench_two_ranks_prints_one_aggregate_line(config, extra):
    """Strong scaling: C3's slots / pool (1024 requests, here 64 slots so two
    ranks fit one GPU) and C5's 4M rows are split over the ranks. Weak scaling:
    C2 (the default) runs one GPU's workload per rank."""
    env = dict(os.environ, DUCHESS_BENCH_BACKEND="gloo")
    if config == "c5":
        env["DUCHESS_C5_ROWS"] = str(1 << 20)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py",
           "--gpus", "2", "--config", config, "--steps", "3", "--warmup", "3",
           "--e2e-steps", "2", "--no-cpu-baseline"] + extra
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    out = json.loads(lines[0])
    assert out["n_gpus"] == 2 and out["steps"] == 3 and out["value"] > 0
    assert out["gpu_launches"] > 0
    assert out["scaling"] == ("weak" if config == "c2" else "strong")
    if config == "c5":
        assert out["config"]["rows"] == 1 << 20 and out["config"]["rows_per_gpu"] == 1 << 19
        assert out["allreduce"]["backend"] == "gloo"
    elif config == "c2":
        assert out["config"]["slots_per_gpu"] == 64 and out["config"]["requests"] == 128
    else:
        assert out["config"]["slots_per_gpu"] * 2 == out["config"]["requests"]
