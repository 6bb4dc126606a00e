"""Host-side pieces of bench.py that need no GPU: the synthetic C4 fork trace
(the shape SURVEY 8(d) names), the committed traffic captures the roofline
cites, and the CPU reference helpers' output contract."""

import json
import os

import numpy as np

import bench

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c4_fork_trace_shape_and_chain_resolution():
    R, roots, nf = 32, 16, 48
    pos, forks = bench.make_fork_trace(R, roots, nf, 16, 256, seed=31)
    assert pos.shape == (R, roots) and forks.shape == (R, nf, 4)
    assert ((pos >= 16) & (pos <= 2048)).all()
    for r in range(R):
        alive_pos = list(pos[r])
        alive_root = list(range(roots))
        for k in range(nf):
            child, src, root, prefix = (int(v) for v in forks[r, k])
            assert child == roots + k and 0 <= src < roots + k
            assert root == alive_root[src] and root < roots        # chains end at a root
            assert prefix == alive_pos[src]                           # child starts at parent pos
            alive_pos.append(prefix)
            alive_root.append(root)
    pos2, forks2 = bench.make_fork_trace(R, roots, nf, 16, 256, seed=31)
    assert np.array_equal(pos, pos2) and np.array_equal(forks, forks2)


def test_traffic_captures_cited_by_the_roofline_exist():
    r32, src32 = bench.k1_traffic_ratio(32)
    r1, src1 = bench.k1_traffic_ratio(1)
    assert src32.endswith("k1_traffic.json") and src1.endswith("k1rows_traffic.json")
    assert 1.0 <= r32 < 1.02 and 1.0 <= r1 < 1.02      # no re-reads beyond 2%
    for src in (src32, src1):
        d = json.load(open(os.path.join(ROOT, src)))
        assert d["dram_bytes"] == d["dram_read_bytes"] + d["dram_write_bytes"]


def test_cpu_reference_helpers_report_value_unit_cores_kind():
    cb = bench.cpu_c3tc(n=256, reps=1)
    assert cb["value"] > 0 and cb["unit"] == "branch-steps/s" and cb["kind"] == "port"
    assert cb["cores"] >= 1 and "sample" in cb


def test_serving_plan_weak_c2_strong_c3():
    """N > 1: C2 (the default) keeps one GPU's workload per rank (weak
    scaling, each rank its own share of an N-times pool); the C3 variants split
    BASELINE configs[2]'s 1024 requests and pool over the ranks (strong)."""
    import bench
    for world in (1, 2, 4, 8):
        shares, slots = [], []
        for rank in range(world):
            R, (lo, hi), pool = bench.serving_plan("c2", world, rank)
            assert R == bench.CONFIGS["c2"]["R"] and pool == bench.CONFIGS["c2"]["pool"] * world
            shares.append((lo, hi))
            slots.append(R)
        assert shares[0][0] == 0 and shares[-1][1] == pool
        assert all(a[1] == b[0] for a, b in zip(shares, shares[1:]))
        for name in bench.STRONG_SCALED:
            got = [bench.serving_plan(name, world, r) for r in range(world)]
            assert sum(R for R, _, _ in got) == bench.CONFIGS[name]["R"]
            assert got[0][1][0] == 0 and got[-1][1][1] == bench.CONFIGS[name]["pool"]
