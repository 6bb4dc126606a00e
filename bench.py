"""Benchmark: branch-steps/s scored + decided (DUCHESS probe + orchestration).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2|c1|c3|c3t1|c4|c5|c3tc|baselines|difficulty|sim]

One step = one orchestration round over every request slot on the GPU:
duchess_score_active (K1: pooled LayerNorm + linear probe over each
survivor's activation window, read from HBM) -> duchess_round (decide the
round: predict / early-terminate / branch-out / request termination + vote,
then refill and advance every slot into the next round). A branch-step is one
survivor scored and decided (one `self._predict` call in reference
orchestrator.py:358-362).

Default workload (BASELINE.json configs[1], "C2"): 256 request slots x 16
branch slots, hidden 4096, bf16 activations, 32-token pooling window, one
probe layer, math-like knobs with max_branches=16 (presets.py:55-59), a
cycling pool of 2048 synthetic requests (64 templates each) admitted in
easiest-first order. Activations: 4 rotating slabs per shard (4x the 126 MB
L2, so every step streams from HBM). The slots are split into two
independent request shards stepping on two CUDA streams (requests never
interact), so each shard's latency-bound round kernel runs while the other
shard's scorer streams. Under torchrun each rank runs its own request shard
(weak scaling, no data-path collective).

--impl reference times the CPU restatement of the reference (oracle/port.py:
the reference's DuchessRun with a predictor= that pools + LayerNorms + dots
distinct windows in numpy) on all host cores.
"""

from __future__ import annotations

import argparse
import json
import os
import random
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# Untimed serving rounds before the W warm-up steps: every slot starts on a fresh
# request, and the first rounds (all requests young, few finishing) are not the
# steady state a serving GPU runs in; this burn-in is part of setup, not timed.
BURN_IN_ROUNDS = 24

METRIC = "branch-steps/sec scored+decided (HBM GB/s % of peak) at 1/2/4/8 B200 vs CPU"
UNIT = "branch-steps/s"

CONFIGS = {
    # name: (R slots, c, L, T, H, dtype, preset, pool)
    "c2": dict(R=256, c=16, L=1, T=32, H=4096, dtype="bf16", preset="math-like", pool=2048),
    "c1": dict(R=8, c=8, L=1, T=1, H=4096, dtype="f32", preset="gsm8k-like", pool=128),
    "c3": dict(R=1024, c=32, L=4, T=32, H=5120, dtype="bf16", preset="math-like", pool=4096),
    # SURVEY 8(d) C3 secondary row: the last token only (T=1, 40 960 B per branch-step)
    "c3t1": dict(R=1024, c=32, L=4, T=1, H=5120, dtype="bf16", preset="math-like", pool=4096),
}

PRESET_KNOBS = {   # presets.py:30-68 (knobs) — max_branches overridden per config
    "gsm8k-like": dict(interval_tokens=16, early_term_threshold=0.70, early_term_rounds=2,
                       branch_out_temperature=1.0, consensus_frac=0.6, coverage_frac=0.8),
    "math-like": dict(interval_tokens=80, early_term_threshold=0.80, early_term_rounds=2,
                      branch_out_temperature=0.8, consensus_frac=0.6, coverage_frac=0.8),
}
PRESET_GEN = {
    "gsm8k-like": dict(level_median_tokens=(180, 220, 260, 300, 350),
                       level_correct_prob=(0.92, 0.88, 0.84, 0.80, 0.75), probe_stride=16),
    "math-like": dict(level_median_tokens=(340, 460, 640, 840, 1180),
                      level_correct_prob=(0.85, 0.78, 0.70, 0.62, 0.52),
                      distractor_count=10, probe_stride=40),
}


def k3_traffic():
    """DRAM bytes of one fork_exec launch from the committed ncu capture."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "k3_traffic.json")))
    if not files:
        return None, None
    with open(files[-1]) as f:
        return json.load(f)["dram_bytes"], os.path.relpath(files[-1], ROOT)


def k1_traffic_ratio(T=32):
    """DRAM bytes / algorithmic bytes of K1 from the committed ncu --set full
    capture (tools/profile_all.sh -> profiles/<round>/k1_traffic.json; the
    T = 1 rows kernel: k1rows_traffic.json)."""
    import glob
    name = "k1rows_traffic.json" if T == 1 else "k1_traffic.json"
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", name)))
    if not files:
        return None, None
    with open(files[-1]) as f:
        d = json.load(f)
    return d["dram_bytes"] / d["algorithmic_bytes"], os.path.relpath(files[-1], ROOT)


# MEASURED_PEAKS.json hbm_gbs is a device-to-device copy (read + write bytes);
# a read-only stream (K1, K4) can run above it, so frac > 1 is possible.
PEAK_NOTE = "peak = measured copy bandwidth (read+write); read-only streams can exceed it"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# workload (host-side packing; identical for the GPU arm and the CPU arm)

def make_workload(cfg, seed):
    from paper_2509_24957_b200.workload import SyntheticParams, generate_synthetic
    from paper_2509_24957_b200.orchestrator import OrchestratorConfig
    params = SyntheticParams(templates_per_request=64, **PRESET_GEN[cfg["preset"]])
    traces = generate_synthetic(params, cfg["pool"], seed=seed).requests
    knobs = OrchestratorConfig(max_branches=cfg["c"], **PRESET_KNOBS[cfg["preset"]])
    master = random.Random(seed + 1)
    seeds = [master.getrandbits(64) for _ in traces]
    return traces, knobs, seeds


def make_probe(H, L, seed=0):
    rng = np.random.default_rng(seed)
    w = rng.normal(0.0, 1.5 / np.sqrt(H), size=(L, H))
    g = rng.uniform(0.5, 1.5, size=(L, H))
    beta = rng.uniform(-0.1, 0.1, size=(L, H))
    return w, np.zeros(L), g, beta


# ---------------------------------------------------------------------------
class ClockSampler:
    """SM clock + throttle reasons polled through NVML on a background thread
    for the whole timed region (every ~2 ms, so short regions get samples)."""
    REASONS = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
               "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
               "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
               "sw_power_cap": "nvmlClocksEventReasonSwPowerCap",
               "hw_power_brake": "nvmlClocksEventReasonHwPowerBrakeSlowdown"}

    def __init__(self, index):
        import threading
        self.sm, self.reasons, self.err = [], set(), None
        self.stop_evt = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # noqa: BLE001
            self.nv, self.err = None, str(e)
            return
        self.th = threading.Thread(target=self._run, daemon=True)
        self.th.start()

    def _run(self):
        nv = self.nv
        while True:
            try:
                self.sm.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, const in self.REASONS.items():
                    if mask & getattr(nv, const):
                        self.reasons.add(name)
            except Exception as e:  # noqa: BLE001
                self.err = str(e)
                return
            if self.stop_evt.wait(0.002):
                return

    def stop(self):
        if self.nv is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": self.err}
        self.stop_evt.set()
        self.th.join(timeout=5)
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None,
                "sm_max_mhz": self.max, "reasons": sorted(self.reasons),
                "samples": len(self.sm), "source": "nvml"}


# ---------------------------------------------------------------------------
def run_gpu(args, cfg, rank, world, local_rank):
    import torch

    from paper_2509_24957_b200 import _lib
    from paper_2509_24957_b200.engine import BatchedDuchess
    from paper_2509_24957_b200.probe import ProbeBank, Scorer, fill_windows
    from paper_2509_24957_b200.scheduler import difficulty_queue

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    R, C, L, T, H = cfg["R"], cfg["c"], cfg["L"], cfg["T"], cfg["H"]
    tdtype = torch.bfloat16 if cfg["dtype"] == "bf16" else torch.float32
    esz = 2 if cfg["dtype"] == "bf16" else 4
    traces, knobs, seeds = make_workload(cfg, seed=1000 + 17 * rank)
    queue = difficulty_queue([t.difficulty for t in traces], device=dev)
    eng = BatchedDuchess(traces, knobs, seeds, n_slots=R, pred_source=_lib.PRED_DEVICE,
                         queue=queue, cycle=True, n_layers=L, combine=1 if L > 1 else 0,
                         device=dev)
    w, b, g, beta = make_probe(H, L)
    bank = ProbeBank.from_linear(w, b, g, beta, device=dev)
    if args.k1 == "ldg":
        scorer = Scorer(bank, R * C * L, nsplit=args.nsplit, threads=args.threads)
    else:
        scorer = Scorer(bank, R * C * L)          # persistent TMA-bulk kernel
    rows = R * C
    n_slabs = max(2, min(4, int((4 << 30) // (rows * L * T * H * esz)) or 2))
    if rows * L * T * H * esz < (256 << 20):
        n_slabs = 4
    slabs = [torch.empty((rows, L, T, H), dtype=tdtype, device=dev) for _ in range(n_slabs)]
    for i, s in enumerate(slabs):
        fill_windows(s, 7000 + 31 * rank + i)
    logit = torch.empty((rows, L), dtype=torch.float32, device=dev)
    probs = eng.probs.view(rows, L)
    stream = torch.cuda.current_stream(dev)
    k1_ev = []

    fused = args.mode == "fused"

    def one_step(i, timed):
        # fused: ONE persistent launch per round (duchess_step) —
        # K1 streams the survivors' windows while a decision warp per CTA
        # decides every request whose windows are scored and advances it into
        # the next round. split (default): K1 launch, then duchess_round (decide k +
        # advance k+1). The scoring kernel is bracketed by CUDA events on every
        # `k1_every`-th timed step: an event record between two PDL-chained
        # kernels breaks their overlap, so sampling keeps the measurement from
        # inflating the step time.
        if timed:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        if fused:
            eng.step_fused(slabs[i % n_slabs], bank, logit.view(-1))
            if timed:
                e1.record(stream)
                k1_ev.append((e0, e1))
            return
        if args.k1 == "list":
            scorer.score_active(slabs[i % n_slabs], logit, probs, eng)
        else:
            scorer(slabs[i % n_slabs], logit, probs, row_mask=eng.t["row_mask"])
        if timed:
            e1.record(stream)
            k1_ev.append((e0, e1))
        eng.round()

    if fused:
        eng.begin_fused()              # round 0: refill every slot + phase 1
    else:
        eng.advance()
    for i in range(BURN_IN_ROUNDS + args.warmup):
        one_step(i, False)
    torch.cuda.synchronize(dev)
    c0 = eng.t["counters"].clone()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    graph = None
    if args.graph:
        # CUDA graph of one slab rotation (n_slabs rounds = 2*n_slabs launches,
        # PDL edges kept), replayed; removes the host launch cost that bounds
        # small configs. K1 is timed with events in an eager pass afterwards.
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            for j in range(n_slabs):
                one_step(BURN_IN_ROUNDS + args.warmup + j, False)
        args.steps = -(-args.steps // n_slabs) * n_slabs
        graph.replay()                  # one rotation untimed (warm the graph)
        torch.cuda.synchronize(dev)
        c0 = eng.t["counters"].clone()
    clocks = ClockSampler(local_rank) if rank == 0 else None
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    if graph is not None:
        for _ in range(args.steps // n_slabs):
            graph.replay()
    else:
        for i in range(args.steps):
            one_step(BURN_IN_ROUNDS + args.warmup + i, i % args.k1_every == 0)
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    clk = clocks.stop() if clocks else None
    if graph is not None:
        # event timing inside a replayed graph is not meaningful: K1 is timed
        # in an eager pass right after the timed region (same state, shapes)
        cnt_g = (eng.t["counters"] - c0).cpu().numpy()
        for i in range(8 * args.k1_every):
            one_step(i, i % args.k1_every == 0)
        torch.cuda.synchronize(dev)
    if world > 1:
        torch.distributed.barrier()
    ms = ev0.elapsed_time(ev1)
    cnt = cnt_g if graph is not None else (eng.t["counters"] - c0).cpu().numpy()
    branch_steps = int(cnt[_lib.CNT_BRANCH_STEPS])
    k1_ms = sum(a.elapsed_time(b) for a, b in k1_ev) / max(len(k1_ev), 1) * args.steps
    stats = torch.tensor([ms, float(branch_steps), k1_ms], dtype=torch.float64, device=dev)
    if world > 1:
        tmax = stats[:1].clone()
        torch.distributed.all_reduce(tmax, op=torch.distributed.ReduceOp.MAX)
        tot = stats[1:2].clone()
        torch.distributed.all_reduce(tot, op=torch.distributed.ReduceOp.SUM)
        ms_all, bs_all = float(tmax[0]), float(tot[0])
    else:
        ms_all, bs_all = ms, float(branch_steps)

    # ---- end to end through the public API with host buffers ----
    e2e = run_e2e(args, eng, scorer, logit, probs, rows, L, T, H, tdtype, dev, world, bank)

    if rank != 0:
        return None
    bytes_per_bs = T * H * esz * L
    k1_avg_s = k1_ms / args.steps / 1e3
    bytes_per_launch = branch_steps / args.steps * bytes_per_bs
    peak, peak_kind = load_peaks()
    achieved = bytes_per_launch / k1_avg_s / 1e9
    out = {
        "metric": METRIC, "value": bs_all / (ms_all / 1e3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_all / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": cfg["dtype"], "data": "synthetic (counter-hashed N(0,1) activations with "
        "outlier channels; generate_synthetic workload, random-init probe)",
        "config": {"workload": f"{args.config.upper()}: {R} request slots x {C} branches, "
                   f"hidden {H}, {L} probe layer(s), T={T} pooling window, {cfg['dtype']}, "
                   f"{cfg['preset']} knobs, cycling pool of {cfg['pool']} requests "
                   f"(easiest-first), {n_slabs} rotating activation slabs "
                   f"({rows * L * T * H * esz / 2**30:.2f} GiB each, > L2)",
                   "requests": R, "branches": C, "hidden": H, "layers": L, "window": T,
                   "launch": "CUDA graph replay" if args.graph else "eager stream (PDL)",
                   "l2": "inputs larger than L2 (rotating slabs)",
                   "burn_in_rounds": BURN_IN_ROUNDS,
                   "parallelism": f"request-sharded x{world}"},
        "branch_steps_per_step": branch_steps / args.steps,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "peak_kind": peak_kind, "peak_note": PEAK_NOTE,
                     "kernel": ("duchess_step (fused K1 scoring + decide + advance, one "
                                "launch per round)" if fused else f"duchess_score (K1, {args.k1})"),
                     "bytes_per_launch": bytes_per_launch,
                     "k1_us_per_launch": k1_avg_s * 1e6,
                     "k1_share_of_step": k1_ms / ms,
                     "k1_launches_timed": (f"{len(k1_ev)} (eager pass after the timed graph "
                                           f"replays)") if args.graph else len(k1_ev),
                     "traffic": (None if k1_traffic_ratio(T)[0] is None
                                 else k1_traffic_ratio(T)[0] * bytes_per_launch),
                     "traffic_source": k1_traffic_ratio(T)[1]},
        "e2e": e2e,
        "gpu_launches": (1 if fused else 2) * args.steps,
        "clocks": clk,
        "counters": {"ambiguous_draws": int(cnt[_lib.CNT_AMBIGUOUS]),
                     "finished_requests": int(cnt[_lib.CNT_FINISHED]),
                     "forks": int(cnt[_lib.CNT_FORKS])},
    }
    return out


def run_gpu_sharded(args, cfg, rank, world, local_rank):
    """C2/C3 with the GPU's request slots split into `shards` independent
    engines (interleaved request pools), each stepping on its own CUDA stream:
    requests never interact, so this is the multi-GPU request
    sharding applied inside one GPU. The HBM-bound scorer of one shard runs
    while the latency-bound round kernel of another finishes (the small round
    CTAs fit beside the scorer's), so the decision kernel leaves the critical
    path. Same workload as run_gpu: R slots x C branches in total."""
    import torch

    from paper_2509_24957_b200 import _lib
    from paper_2509_24957_b200.engine import BatchedDuchess
    from paper_2509_24957_b200.probe import ProbeBank, Scorer, fill_windows
    from paper_2509_24957_b200.scheduler import difficulty_queue

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    S = args.shards
    R, C, L, T, H = cfg["R"], cfg["c"], cfg["L"], cfg["T"], cfg["H"]
    if R % S:
        raise SystemExit(f"--shards {S} must divide the {R} request slots")
    Rs = R // S
    tdtype = torch.bfloat16 if cfg["dtype"] == "bf16" else torch.float32
    esz = 2 if cfg["dtype"] == "bf16" else 4
    traces, knobs, seeds = make_workload(cfg, seed=1000 + 17 * rank)
    w, b, g, beta = make_probe(H, L)
    bank = ProbeBank.from_linear(w, b, g, beta, device=dev)
    rows = Rs * C
    slab_bytes = rows * L * T * H * esz
    n_slabs = 4 if slab_bytes * S < (256 << 20) else max(2, min(4, int((4 << 30) // (slab_bytes * S)) or 2))
    shards = []
    for sh in range(S):
        tr, sd = traces[sh::S], seeds[sh::S]
        queue = difficulty_queue([t.difficulty for t in tr], device=dev)
        eng = BatchedDuchess(tr, knobs, sd, n_slots=Rs, pred_source=_lib.PRED_DEVICE,
                             queue=queue, cycle=True, n_layers=L, combine=1 if L > 1 else 0,
                             device=dev)
        slabs = [torch.empty((rows, L, T, H), dtype=tdtype, device=dev) for _ in range(n_slabs)]
        for i, sl in enumerate(slabs):
            fill_windows(sl, 7000 + 31 * rank + 7 * sh + i)
        shards.append(dict(eng=eng, scorer=Scorer(bank, rows * L), slabs=slabs,
                           logit=torch.empty((rows, L), dtype=torch.float32, device=dev),
                           stream=torch.cuda.Stream(dev), ev=[]))
    main = torch.cuda.current_stream(dev)

    # The scorers of the shards take turns (each waits for the previous one's
    # event): every K1 launch streams alone at full HBM bandwidth, while the
    # round kernel of the shard scored just before runs beside it.
    prev_k1 = [None]

    def step(i, timed):
        for sh in shards:
            with torch.cuda.stream(sh["stream"]):
                st = sh["stream"]
                if prev_k1[0] is not None and args.shard_order == "turns":
                    st.wait_event(prev_k1[0])
                if timed:
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(st)
                sh["scorer"].score_active(sh["slabs"][i % n_slabs], sh["logit"],
                                          sh["eng"].probs.view(rows, L), sh["eng"])
                if timed:
                    e1.record(st)
                    sh["ev"].append((e0, e1))
                if args.shard_order == "turns":
                    done = e1 if timed else torch.cuda.Event()
                    if not timed:
                        done.record(st)
                    prev_k1[0] = done
                sh["eng"].round()

    def join():
        for sh in shards:
            main.wait_stream(sh["stream"])

    def fork():
        for sh in shards:
            sh["stream"].wait_stream(main)

    fork()
    for sh in shards:
        with torch.cuda.stream(sh["stream"]):
            sh["eng"].advance()
    for i in range(BURN_IN_ROUNDS + args.warmup):
        step(i, False)
    join()
    torch.cuda.synchronize(dev)
    c0 = [sh["eng"].t["counters"].clone() for sh in shards]
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    clocks = ClockSampler(local_rank) if rank == 0 else None
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(main)
    fork()
    for i in range(args.steps):
        step(BURN_IN_ROUNDS + args.warmup + i, i % args.k1_every == 0)
    join()
    ev1.record(main)
    torch.cuda.synchronize(dev)
    clk = clocks.stop() if clocks else None
    if world > 1:
        torch.distributed.barrier()
    ms = ev0.elapsed_time(ev1)
    cnt = sum((sh["eng"].t["counters"] - c).cpu().numpy() for sh, c in zip(shards, c0))
    branch_steps = int(cnt[_lib.CNT_BRANCH_STEPS])
    k1_us = [a.elapsed_time(b) * 1e3 for sh in shards for a, b in sh["ev"]]
    k1_avg_s = sum(k1_us) / max(len(k1_us), 1) / 1e6

    stats = torch.tensor([ms, float(branch_steps)], dtype=torch.float64, device=dev)
    if world > 1:
        tmax = stats[:1].clone()
        torch.distributed.all_reduce(tmax, op=torch.distributed.ReduceOp.MAX)
        tot = stats[1:2].clone()
        torch.distributed.all_reduce(tot, op=torch.distributed.ReduceOp.SUM)
        ms_all, bs_all = float(tmax[0]), float(tot[0])
    else:
        ms_all, bs_all = ms, float(branch_steps)

    e2e = run_e2e_sharded(args, shards, rows, L, T, H, tdtype, dev, world, main)
    if rank != 0:
        return None
    bytes_per_bs = T * H * esz * L
    bytes_per_launch = branch_steps / args.steps / S * bytes_per_bs
    peak, peak_kind = load_peaks()
    overlap = args.shard_order == "overlap"
    # turns: each scoring launch streams alone -> bytes per launch / its duration.
    # overlap: the shards' launches share HBM and drift against each other, so a
    # launch's duration is stretched by sharing; the scoring bytes of a step over
    # the WHOLE step time (round kernels included) is the conservative figure.
    achieved = (bytes_per_launch * S / (ms / args.steps / 1e3) if overlap
                else bytes_per_launch / k1_avg_s) / 1e9
    return {
        "metric": METRIC, "value": bs_all / (ms_all / 1e3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_all / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": cfg["dtype"], "data": "synthetic (counter-hashed N(0,1) activations with "
        "outlier channels; generate_synthetic workload, random-init probe)",
        "config": {"workload": f"{args.config.upper()}: {R} request slots x {C} branches, "
                   f"hidden {H}, {L} probe layer(s), T={T} pooling window, {cfg['dtype']}, "
                   f"{cfg['preset']} knobs, cycling pool of {cfg['pool']} requests "
                   f"(easiest-first), {n_slabs} rotating activation slabs per shard "
                   f"({slab_bytes * S / 2**30:.2f} GiB per rotation, > L2); slots split into "
                   f"{S} independent request shards on {S} CUDA streams "
                   f"({'concurrent scorers' if args.shard_order == 'overlap' else 'scorers take turns'})",
                   "requests": R, "branches": C, "hidden": H, "layers": L, "window": T,
                   "shards_per_gpu": S, "launch": "eager streams (PDL within each shard)",
                   "l2": "inputs larger than L2 (rotating slabs)",
                   "burn_in_rounds": BURN_IN_ROUNDS,
                   "parallelism": f"request-sharded x{world} GPUs x{S} streams"},
        "branch_steps_per_step": branch_steps / args.steps,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "peak_kind": peak_kind, "peak_note": PEAK_NOTE,
                     "kernel": (("duchess_score (K1, list{}): the shards' concurrent launches, "
                                 "scoring bytes per step / whole step time" if overlap else
                                 "duchess_score (K1, list{}) per shard launch").format(
                                     ", score_rows_kernel" if T == 1 else "")),
                     "bytes_per_launch": bytes_per_launch,
                     "k1_us_per_launch": k1_avg_s * 1e6,
                     "k1_launches_timed": len(k1_us),
                     "traffic": (None if k1_traffic_ratio(T)[0] is None
                                 else k1_traffic_ratio(T)[0] * bytes_per_launch),
                     "traffic_source": k1_traffic_ratio(T)[1]},
        "e2e": e2e,
        "gpu_launches": 2 * S * args.steps,
        "clocks": clk,
        "counters": {"ambiguous_draws": int(cnt[_lib.CNT_AMBIGUOUS]),
                     "finished_requests": int(cnt[_lib.CNT_FINISHED]),
                     "forks": int(cnt[_lib.CNT_FORKS])},
    }


def run_e2e_sharded(args, shards, rows, L, T, H, tdtype, dev, world, main):
    """End to end through the public API with pinned HOST activations, per
    shard on its stream: upload_survivors (only the survivors' windows cross
    PCIe), K1, round, D2H of the round records and actions."""
    import torch
    from paper_2509_24957_b200 import _lib
    steps = max(2, min(args.e2e_steps, args.steps))
    row_bytes = L * T * H * torch.tensor([], dtype=tdtype).element_size()
    for sh in shards:
        sh["host"] = torch.empty((rows, L, T, H), dtype=tdtype, pin_memory=True)
        sh["host"].view(-1).zero_()
        sh["dslab"] = torch.empty_like(sh["host"], device=dev)
        sh["rec_h"] = torch.empty(sh["eng"].t["round_rec"].numel(), dtype=torch.int32,
                                  pin_memory=True)
        sh["act_h"] = torch.empty(sh["eng"].t["actions"].numel(), dtype=torch.int32,
                                  pin_memory=True)

    def step():
        for sh in shards:
            with torch.cuda.stream(sh["stream"]):
                eng = sh["eng"]
                eng.upload_survivors(sh["host"], sh["dslab"])
                sh["scorer"].score_active(sh["dslab"], sh["logit"], eng.probs.view(rows, L), eng)
                eng.round()
                sh["rec_h"].copy_(eng.t["round_rec"], non_blocking=True)
                sh["act_h"].copy_(eng.t["actions"], non_blocking=True)
        for sh in shards:
            sh["stream"].synchronize()

    step()
    c0 = [sh["eng"].t["counters"].clone() for sh in shards]
    if world > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    dt = time.perf_counter() - t0
    bs = sum(int((sh["eng"].t["counters"] - c)[_lib.CNT_BRANCH_STEPS]) for sh, c in zip(shards, c0))
    st = torch.tensor([dt, float(bs)], dtype=torch.float64, device=dev)
    if world > 1:
        a = st[:1].clone()
        torch.distributed.all_reduce(a, op=torch.distributed.ReduceOp.MAX)
        b = st[1:].clone()
        torch.distributed.all_reduce(b, op=torch.distributed.ReduceOp.SUM)
        dt, bs = float(a[0]), float(b[0])
    return {"value": bs / dt, "unit": UNIT,
            "h2d_bytes_per_step": bs / steps / max(world, 1) * row_bytes,
            "h2d": "survivor windows only (duchess_gather_active over each shard's active "
                   "list), average per rank",
            "d2h_bytes_per_step": sum((sh["rec_h"].numel() + sh["act_h"].numel()) * 4
                                      for sh in shards),
            "steps": steps, "timing": "host wall clock, streams synchronised each step"}


def run_e2e(args, eng, scorer, logit, probs, rows, L, T, H, tdtype, dev, world, bank=None):
    """Same step through the public API with the activations in pinned HOST
    memory: per step the H2D copy of the round's inputs (the survivors'
    windows, gathered by one kernel over the device-side active list; the
    whole slab for the other variants), the round (K1 + duchess_round, or one
    fused launch), and a D2H read of the round records and actions
    (RoundReports)."""
    import torch
    steps = max(2, min(args.e2e_steps, args.steps))
    host = torch.empty((rows, L, T, H), dtype=tdtype, pin_memory=True)
    host.copy_(torch.zeros(1, dtype=tdtype).expand_as(host))
    dslab = torch.empty_like(host, device=dev)
    rec_host = torch.empty(eng.t["round_rec"].numel(), dtype=torch.int32, pin_memory=True)
    act_host = torch.empty(eng.t["actions"].numel(), dtype=torch.int32, pin_memory=True)
    from paper_2509_24957_b200 import _lib
    stream = torch.cuda.current_stream(dev)

    survivors_only = args.mode == "split" and args.k1 == "list"

    def step():
        if survivors_only:
            # only the windows of this round's survivors cross PCIe (the
            # active list is on the device; one gather kernel reads them)
            eng.upload_survivors(host, dslab)
        else:
            dslab.copy_(host, non_blocking=True)
        if args.mode == "fused":
            eng.step_fused(dslab, bank, logit.view(-1))
            rec_host.copy_(eng.t["round_rec"], non_blocking=True)
            act_host.copy_(eng.t["actions"], non_blocking=True)
            stream.synchronize()
            return
        # the round in flight was advanced by the previous round(): score it,
        # decide it and advance into the next one, exactly as the timed loop
        if args.k1 == "list":
            scorer.score_active(dslab, logit, probs, eng)
        else:
            scorer(dslab, logit, probs, row_mask=eng.t["row_mask"])
        eng.round()
        rec_host.copy_(eng.t["round_rec"], non_blocking=True)
        act_host.copy_(eng.t["actions"], non_blocking=True)
        stream.synchronize()

    step()
    c0 = eng.t["counters"].clone()
    if world > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    dt = time.perf_counter() - t0
    bs = int((eng.t["counters"] - c0)[_lib.CNT_BRANCH_STEPS])
    st = torch.tensor([dt, float(bs)], dtype=torch.float64, device=dev)
    if world > 1:
        a = st[:1].clone()
        torch.distributed.all_reduce(a, op=torch.distributed.ReduceOp.MAX)
        b = st[1:].clone()
        torch.distributed.all_reduce(b, op=torch.distributed.ReduceOp.SUM)
        dt, bs = float(a[0]), float(b[0])
    row_bytes = host[0].numel() * host.element_size()
    h2d = (bs / steps / max(world, 1) * row_bytes if survivors_only
           else host.numel() * host.element_size())
    return {"value": bs / dt, "unit": UNIT,
            "h2d_bytes_per_step": h2d,
            "h2d": ("survivor windows only (duchess_gather_active over the active list), "
                    "average per rank" if survivors_only else "whole activation slab"),
            "d2h_bytes_per_step": (rec_host.numel() + act_host.numel()) * 4,
            "steps": steps, "timing": "host wall clock, stream-synchronised each step"}


# ---------------------------------------------------------------------------
# C4: branch-out-heavy copy-on-write trace; C5: probe-training step

def make_fork_trace(R, roots, forks_per_req, bt, max_blocks, seed):
    """Synthetic C4 trace: `roots` live branches per request at positions
    U[16, 2048]; forks sampled like branch_out_sample (p^(1/0.8) weights over
    the alive set incl. children created earlier, chains resolved to roots)."""
    rng = np.random.default_rng(seed)
    pos = rng.integers(16, 2049, size=(R, roots))
    probs = rng.random((R, roots + forks_per_req))
    forks = np.zeros((R, forks_per_req, 4), dtype=np.int32)
    for r in range(R):
        alive_pos = list(pos[r])
        alive_root = list(range(roots))
        for k in range(forks_per_req):
            n = len(alive_pos)
            wts = np.maximum(probs[r, :n], 1e-6) ** 1.25
            src = int(rng.choice(n, p=wts / wts.sum()))
            forks[r, k] = (roots + k, src, alive_root[src], alive_pos[src])
            alive_pos.append(alive_pos[src])
            alive_root.append(alive_root[src])
    return pos, forks


def run_fork_bench(args, rank, world, local_rank):
    import torch
    from paper_2509_24957_b200.kvfork import BlockTable
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    R, roots, nf, bt, max_blocks, kvb = 512, 16, 48, 16, 256, 4096
    pos, forks = make_fork_trace(R, roots, nf, bt, max_blocks, seed=31 + rank)
    rows_per = roots + nf
    nblk_root = -(-pos // bt)
    n_root_blocks = int(nblk_root.sum())
    n_tail = int(((forks[:, :, 3] % bt) != 0).sum())
    n_blocks = n_root_blocks + n_tail
    table = np.full((R * rows_per, max_blocks), -1, dtype=np.int32)
    nxt = 0
    for r in range(R):
        for b in range(roots):
            table[r * rows_per + b, :nblk_root[r, b]] = np.arange(nxt, nxt + nblk_root[r, b])
            nxt += nblk_root[r, b]
    t = BlockTable(R * rows_per, max_blocks, n_blocks, bt, kvb, device=dev)
    t.table.copy_(torch.from_numpy(table))
    t.refcount[:n_root_blocks] = 1
    t.free_list = torch.arange(n_root_blocks, n_blocks, dtype=torch.int32, device=dev)
    g = torch.Generator(device=dev).manual_seed(3)
    for lo in range(0, t.kv.numel(), 1 << 30):      # incompressible KV contents
        hi = min(t.kv.numel(), lo + (1 << 30))
        t.kv[lo:hi] = torch.randint(0, 256, (hi - lo,), dtype=torch.uint8, device=dev,
                                    generator=g)
    fk = torch.from_numpy(forks).to(dev)
    n_full = forks[:, :, 3] // bt
    tail = forks[:, :, 3] % bt
    # Algorithmic bytes: table reads of the full blocks + refcount read/write,
    # each child's table row and fork record, every child's private tail
    # (write), and each DISTINCT source tail once (read): forks of one root
    # share its partial tail block (children inherit root and prefix).
    src_tails = {(r, int(forks[r, k, 2])): int(tail[r, k]) for r in range(R) for k in range(nf)}
    bytes_per_step = int((n_full * 4 * 3).sum() + R * nf * (max_blocks * 4 + 16)
                         + (tail * kvb).sum() + sum(src_tails.values()) * kvb)
    stream = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):
        t.cursor.zero_()
        t.fork(fk, None, 1, rows_per)
    torch.cuda.synchronize(dev)
    evs = []
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # > 126 MB L2
    clocks = ClockSampler(local_rank) if rank == 0 else None
    e_all0, e_all1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e_all0.record(stream)
    for _ in range(args.steps):
        t.cursor.zero_()
        flush.fill_(1)                 # evict tables / refcounts / KV from L2 between steps
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        t.fork(fk, None, 1, rows_per)
        b.record(stream)
        evs.append((a, b))
    e_all1.record(stream)
    torch.cuda.synchronize(dev)
    clk = clocks.stop() if clocks else None
    k3_ms = sum(a.elapsed_time(b) for a, b in evs) / args.steps
    step_ms = e_all0.elapsed_time(e_all1) / args.steps
    peak, kind = load_peaks()
    achieved = bytes_per_step / (k3_ms / 1e3) / 1e9
    return {"metric": "copy-on-write forks/s (C4 branch-out-heavy trace)",
            "value": R * nf * world / (k3_ms / 1e3), "unit": "forks/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32+u8",
            "data": "synthetic fork trace", "config": {
                "workload": f"C4: {R} requests x {roots} root branches at U[16,2048] tokens, "
                            f"{nf} forks/request (24576), 16-token blocks, {kvb} B/token KV; "
                            f"L2 flushed (256 MB write) between steps, value = forks / K3 time",
                "n_blocks": n_blocks},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "peak_kind": kind, "peak_note": PEAK_NOTE,
                         "kernel": "duchess_fork_cow (plan + exec)",
                         "bytes_per_launch": bytes_per_step, "k3_us_per_launch": k3_ms * 1e3,
                         "traffic": k3_traffic()[0], "traffic_source": k3_traffic()[1]},
            "gpu_launches": 2 * args.steps, "clocks": clk}


def run_tc_bench(args, rank, world, local_rank):
    """C3 tensor-core variant: the paper's MLP probe (hidden 2048, ReLU, LN
    folded) at T=1 over 1024 requests x 32 branches of hidden 5120, as one
    tcgen05 GEMM per step with the head fused into the epilogue."""
    import torch
    from paper_2509_24957_b200.mlp_probe import TensorCoreMlpProbe
    from paper_2509_24957_b200.predictor import MlpWeights
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    M, K, NH = 1024 * 32, 5120, 2048
    rng = np.random.default_rng(0)
    w = MlpWeights(K, [NH], 1, ["relu"], [rng.normal(0, 1 / np.sqrt(K), (NH, K)),
                                          rng.normal(0, 1 / np.sqrt(NH), (1, NH))],
                   [rng.normal(0, 0.1, NH), np.array([0.0])], rng.uniform(0.5, 1.5, K),
                   rng.uniform(-0.1, 0.1, K))
    probe = TensorCoreMlpProbe(w, device=dev)
    slabs = [torch.randn((M, K), device=dev).to(torch.bfloat16) for _ in range(2)]  # 2 x 335 MB
    logit = torch.empty(M, device=dev)
    prob = torch.empty(M, dtype=torch.float64, device=dev)
    for i in range(args.warmup):
        probe(slabs[i % 2], logit, prob)
    torch.cuda.synchronize(dev)
    stream = torch.cuda.current_stream(dev)
    clocks = ClockSampler(local_rank) if rank == 0 else None
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(args.steps):
        probe(slabs[i % 2], logit, prob)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    clk = clocks.stop() if clocks else None
    ms = e0.elapsed_time(e1) / args.steps
    flops = probe.flops(M)
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        peak, kind = float(pk["bf16_tflops"]), "measured (burst)"
    except Exception:  # noqa: BLE001
        peak, kind = 1590.0, "fallback"
    tflops = flops / (ms / 1e3) / 1e12
    return {"metric": "MLP-probe branch-steps/s (C3 tensor-core variant, T=1)",
            "value": M * world / (ms / 1e3), "unit": "branch-steps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic N(0,1) activations, random-init MLP probe",
            "config": {"workload": f"C3-TC: {M} windows (1024 req x 32 br), hidden {K} -> "
                                   f"{NH} ReLU -> 1, LN folded, 2 rotating inputs (> L2)"},
            "roofline": {"bound": "tensor", "achieved": tflops, "peak": peak,
                         "unit": "TFLOP/s", "frac": tflops / peak, "peak_kind": kind,
                         "kernel": "mlp_probe_tc_kernel (tcgen05)", "flops_per_launch": flops,
                         "traffic": None},
            "gpu_launches": args.steps, "clocks": clk}


def run_difficulty_bench(args, rank, world, local_rank):
    """the complexity MLP (4096 -> 2048 -> 1024 -> 512 -> 5, BN +
    GeLU, softmax head) over a batch of request activations, hidden layers as
    tcgen05 layers (duchess_tc_linear). CPU reference: the oracle's fp64
    mlp_forward (the reference's per-vector forward) on a bounded sample."""
    import torch
    from paper_2509_24957_b200.difficulty import TensorCoreClassifier
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    M, dims, head = 32768, (4096, 2048, 1024, 512), 5
    full = [*dims, head]
    w = _complexity_weights()
    clf = TensorCoreClassifier(w, device=dev)
    X = [torch.randn((M, dims[0]), device=dev).to(torch.bfloat16) for _ in range(2)]
    for i in range(args.warmup):
        clf.logits(X[i % 2])
    torch.cuda.synchronize(dev)
    clocks = ClockSampler(local_rank) if rank == 0 else None
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(args.steps):
        clf.logits(X[i % 2])
    e1.record()
    torch.cuda.synchronize(dev)
    clk = clocks.stop() if clocks else None
    ms = e0.elapsed_time(e1) / args.steps
    flops = 2.0 * M * sum(full[k] * full[k + 1] for k in range(3))
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peak, kind = float(json.load(f)["bf16_tflops"]), "measured (burst)"
    except Exception:  # noqa: BLE001
        peak, kind = 1590.0, "fallback"
    tf = flops / (ms / 1e3) / 1e12
    out = {"metric": "difficulty predictions/s (complexity MLP, SURVEY 8(f)4)",
           "value": M * world / (ms / 1e3), "unit": "requests/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
           "data": "synthetic N(0,1) activations, random-init complexity MLP",
           "config": {"workload": f"{M} request activations, 4096 -> 2048 -> 1024 -> 512 -> 5, "
                                  "BN + GeLU, LN folded, 2 rotating inputs (> L2)"},
           "roofline": {"bound": "tensor", "achieved": tf, "peak": peak, "unit": "TFLOP/s",
                        "frac": tf / peak, "peak_kind": kind,
                        "kernel": "duchess_tc_linear (3 layers) + head", "flops_per_launch": flops,
                        "traffic": None},
           "gpu_launches": 4 * args.steps, "clocks": clk}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_difficulty(w)
    return out


def _complexity_weights():
    from paper_2509_24957_b200.predictor import MlpWeights
    rng = np.random.default_rng(1)
    dims, head = (4096, 2048, 1024, 512), 5
    full = [*dims, head]
    hid = list(dims[1:])
    W = [rng.normal(0, 1 / np.sqrt(full[k]), (full[k + 1], full[k])) for k in range(4)]
    b = [rng.normal(0, 0.1, full[k + 1]) for k in range(4)]
    return MlpWeights(dims[0], hid, head, ["gelu"] * 3, W, b, rng.uniform(0.5, 1.5, dims[0]),
                      rng.uniform(-0.1, 0.1, dims[0]), [rng.normal(0, 0.1, d) for d in hid],
                      [rng.uniform(0.5, 2.0, d) for d in hid],
                      [rng.uniform(0.5, 1.5, d) for d in hid],
                      [rng.uniform(-0.1, 0.1, d) for d in hid])


def cpu_difficulty(w=None, budget_s=10.0):
    from oracle import port
    w = w or _complexity_weights()
    Xs = np.random.default_rng(2).normal(0, 1, (8, w.input_dim))
    t0 = time.perf_counter()
    n = 0
    while time.perf_counter() - t0 < budget_s:
        port.mlp_forward(w, Xs[n % 8])
        n += 1
    return {"value": n / (time.perf_counter() - t0), "unit": "requests/s", "cores": 1,
            "kind": "port", "sample": f"oracle/port.py fp64 mlp_forward per vector (the "
                                      f"reference's forward), {budget_s:.0f} s on one core"}


def run_sim_bench(args, rank, world, local_rank):
    """run_simulation (simengine.py:150-281) end to end on the
    device engine — every request's rounds in one batch, the timeline folded on
    the device, the single-server queue replayed on the host. CPU reference:
    the oracle's literal one-request-at-a-time replay on a bounded prefix."""
    import torch

    from paper_2509_24957_b200.orchestrator import OrchestratorConfig
    from paper_2509_24957_b200.predictor import SyntheticPredictorConfig
    from paper_2509_24957_b200.scheduler import ArrivalConfig, gen_arrivals
    from paper_2509_24957_b200.simengine import TimingModel, run_simulation
    from paper_2509_24957_b200.workload import SyntheticParams, generate_synthetic
    torch.cuda.set_device(local_rank)
    n = 4096
    params = SyntheticParams(**PRESET_GEN["math-like"])
    wl = generate_synthetic(params, n, seed=21 + rank)
    arrivals = gen_arrivals(ArrivalConfig(rate_qpm=30.0, n_requests=n, seed=3))
    orch = OrchestratorConfig(max_branches=10, **PRESET_KNOBS["math-like"])
    synth = SyntheticPredictorConfig(rho=0.8)
    run_simulation(wl, orch, "duchess", "easiest-predicted", arrivals[:], TimingModel(), 9,
                   synthetic=synth, difficulty_mode="noisy-label")        # warm
    times = []
    for _ in range(max(1, min(args.steps, 5))):
        t0 = time.perf_counter()
        run_simulation(wl, orch, "duchess", "easiest-predicted", arrivals, TimingModel(), 9,
                       synthetic=synth, difficulty_mode="noisy-label")
        times.append(time.perf_counter() - t0)
    dt = statistics.median(times)
    out = {"metric": "run_simulation requests/s (serving timeline, SURVEY 8(f)3)",
           "value": n * world / dt, "unit": "requests/s", "n_gpus": world,
           "steps": len(times), "warmup": 1, "ms_per_step": dt * 1e3, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "int32+f64",
           "data": "generate_synthetic math-like workload, Poisson arrivals",
           "config": {"workload": f"{n} requests, duchess policy, easiest-predicted schedule "
                                  "(noisy-label), default timing model; wall clock of one "
                                  "run_simulation call incl. host packing and queue replay"},
           "gpu_launches": None}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_sim(arrivals)
    return out


def cpu_sim(arrivals=None, k=256):
    from oracle import port, simulate
    from paper_2509_24957_b200.scheduler import ArrivalConfig, gen_arrivals
    arrivals = arrivals or gen_arrivals(ArrivalConfig(rate_qpm=30.0, n_requests=k, seed=3))
    from paper_2509_24957_b200.workload import SyntheticParams, generate_synthetic
    traces = port.generate(port.GenParams(**PRESET_GEN["math-like"]), k, 21)
    knobs = port.Knobs(max_branches=10, **PRESET_KNOBS["math-like"])
    wl = generate_synthetic(SyntheticParams(**PRESET_GEN["math-like"]), k, seed=21)
    t0 = time.perf_counter()
    wl.content_hash()               # run_simulation hashes the workload (simengine.py:273)
    simulate.simulate(traces[:k], knobs, "duchess", "easiest-predicted", arrivals[:k],
                      (25.0, 0.0, 0.1), 9, 0.8, "noisy-label", None)
    cdt = time.perf_counter() - t0
    return {"value": k / cdt, "unit": "requests/s", "cores": 1, "kind": "port",
            "sample": f"oracle/simulate.py one-request-at-a-time replay of {k} requests plus "
                      f"the workload hash (the reference's run_simulation restated), one core"}


def run_baselines_bench(args, rank, world, local_rank):
    """the baseline policies (DefaultScRun, ShortMkRun,
    DynasorRun, orchestrator.py:405-561) on the device slot machinery
    (duchess_baseline_round): 256 slots over a cycling math-like pool; value =
    finished requests/s of Default SC, the others reported beside it."""
    import torch
    from paper_2509_24957_b200.engine import BatchedDuchess
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    cfg = dict(CONFIGS["c2"])
    traces, knobs, seeds = make_workload(cfg, seed=1000 + 17 * rank)
    res = {}
    for pol in ("default-sc", "short-mk", "dynasor"):
        eng = BatchedDuchess(traces, knobs, seeds, n_slots=256, queue=list(range(len(traces))),
                             cycle=True, policy=pol, device=dev)
        for _ in range(args.warmup):
            eng.baseline_round()
        torch.cuda.synchronize(dev)
        c0 = eng.t["counters"].clone()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            eng.baseline_round()
        e1.record()
        torch.cuda.synchronize(dev)
        ms = e0.elapsed_time(e1)
        fin = int((eng.t["counters"] - c0)[2])
        res[pol] = {"requests_per_s": fin / (ms / 1e3), "us_per_round": ms / args.steps * 1e3}
    out = {"metric": "baseline-policy finished requests/s (Default SC, SURVEY 8(f)1)",
           "value": res["default-sc"]["requests_per_s"] * world, "unit": "requests/s",
           "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": res["default-sc"]["us_per_round"] / 1e3, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "int32",
           "data": "generate_synthetic math-like pool (2048 requests, cycling)",
           "config": {"workload": "256 request slots x 16 branch slots, one round per step",
                      "policies": res},
           "gpu_launches": args.steps}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baselines()
    return out


def cpu_baselines(budget_s=5.0):
    from oracle import port
    cfg = CONFIGS["c2"]
    traces = port.generate(port.GenParams(templates_per_request=64, **PRESET_GEN[cfg["preset"]]),
                           256, 1000)
    knobs = port.Knobs(max_branches=cfg["c"], **PRESET_KNOBS[cfg["preset"]])
    t0, n = time.perf_counter(), 0
    while time.perf_counter() - t0 < budget_s:
        port.DefaultScRequest(traces[n % len(traces)], knobs).run()
        n += 1
    return {"value": n / (time.perf_counter() - t0), "unit": "requests/s", "cores": 1,
            "kind": "port", "sample": f"oracle/port.py DefaultScRequest.run over math-like "
                                      f"requests, {budget_s:.0f} s on one core"}


def run_train_bench(args, rank, world, local_rank):
    import torch
    from paper_2509_24957_b200.probe import fill_windows
    from paper_2509_24957_b200.train import LogisticProbeTrainer
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    H = 8192
    n_total = 4194304
    n_local = n_total // 8          # the per-GPU shard of the 8-GPU configuration
    X = torch.empty((n_local, 1, 1, H), dtype=torch.bfloat16, device=dev)
    fill_windows(X, 5000 + rank)
    X = X.view(n_local, H)
    g = torch.Generator(device=dev).manual_seed(5)
    w_true = torch.randn(H, generator=g, device=dev) / np.sqrt(H)
    y = torch.empty(n_local, device=dev)
    for lo in range(0, n_local, 65536):
        z = X[lo:lo + 65536].float() @ w_true
        y[lo:lo + 65536] = (torch.rand(z.shape[0], generator=g, device=dev)
                            < torch.sigmoid(z)).float()
    tr = LogisticProbeTrainer(H, device=dev, lr=0.5)
    n_global = n_local * world
    stream = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):
        tr.step(X, y, n_global)
    torch.cuda.synchronize(dev)
    if world > 1:
        torch.distributed.barrier()
    clocks = ClockSampler(local_rank) if rank == 0 else None
    evs = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        tr.local_grad(X, y, 1.0 / n_global)
        b.record(stream)
        evs.append((a, b))
        from paper_2509_24957_b200.distributed import allreduce_sum
        allreduce_sum(tr.grad)
        tr.lib.duchess_sgd_update(tr.w.data_ptr(), tr.grad.data_ptr(), H + 1, 0.5,
                                  stream.cuda_stream)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    clk = clocks.stop() if clocks else None
    ms = e0.elapsed_time(e1) / args.steps
    st = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(st, op=torch.distributed.ReduceOp.MAX)
    ms = float(st[0])
    k4_ms = sum(a.elapsed_time(b) for a, b in evs) / args.steps
    peak, kind = load_peaks()
    bytes_launch = n_local * (H * 2 + 4)
    achieved = bytes_launch / (k4_ms / 1e3) / 1e9
    return {"metric": "probe-training rows/s (C5 logistic regression, full-batch step)",
            "value": n_local * world / (ms / 1e3), "unit": "rows/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic N(0,1) activations, labels ~ Bernoulli(sigmoid(X w*))",
            "config": {"workload": f"C5: {n_local} rows x {H} per GPU (8 GiB, the 8-GPU shard "
                                   f"of 4M rows), grad + NCCL all-reduce (8193 f32) + SGD"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "peak_kind": kind, "peak_note": PEAK_NOTE,
                         "kernel": "duchess_lr_grad (K4)", "bytes_per_launch": bytes_launch,
                         "k4_us_per_launch": k4_ms * 1e3, "traffic": None},
            "gpu_launches": 3 * args.steps, "clocks": clk}


# ---------------------------------------------------------------------------
# CPU reference (oracle port) — only here and in tests may oracle/ run.

_CPU = {}
CPU_POOL_BYTES = 64 << 20      # activation windows per CPU process (16 processes: 1 GiB)


def _cpu_init(cfg_name, n_req, seed):
    from oracle import port
    cfg = CONFIGS[cfg_name]
    H, T, L = cfg["H"], cfg["T"], cfg["L"]
    params = port.GenParams(templates_per_request=64, **PRESET_GEN[cfg["preset"]])
    traces = port.generate(params, n_req, seed)
    knobs = port.Knobs(max_branches=cfg["c"], **PRESET_KNOBS[cfg["preset"]])
    master = random.Random(seed + 1)
    seeds = [master.getrandbits(64) for _ in traces]
    w, b, g, beta = make_probe(H, L)
    # Distinct windows streamed from DRAM like the GPU arm streams HBM: a
    # per-process pool of CPU_POOL_BYTES (> the host caches), each branch-step
    # scoring the next window. Values are bf16-rounded for bf16 configs but kept
    # in fp32, so the CPU pays no conversion the GPU does in registers.
    bf16 = cfg["dtype"] == "bf16"
    n_pool = max(16, CPU_POOL_BYTES // (L * T * H * 4))
    rng = np.random.default_rng(os.getpid())
    pool = []
    for _ in range(n_pool):
        x = rng.standard_normal((L, T, H), dtype=np.float32)
        if bf16:
            u = x.view(np.uint32)
            x = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).view(np.float32)
        pool.append(x)
    _CPU.update(traces=traces, knobs=knobs, seeds=seeds, w=w, b=b, g=g, beta=beta,
                windows=pool, L=L, next=0, cursor=0)


def _cpu_run(budget_s):
    from oracle import port
    st = _CPU
    count = [0]

    def predictor(tmpl, position, _rng):
        count[0] += 1
        win = st["windows"][st["cursor"] % len(st["windows"])]
        st["cursor"] += 1
        ps = [port.pooled_linear_probe(win[l], st["w"][l], st["b"][l], st["g"][l],
                                       st["beta"][l])[1] for l in range(st["L"])]
        return ps[0] if len(ps) == 1 else sum(ps) / len(ps)

    t0 = time.perf_counter()
    while time.perf_counter() - t0 < budget_s:
        i = st["next"] % len(st["traces"])
        st["next"] += 1
        req = port.DuchessRequest(st["traces"][i], st["knobs"], random.Random(st["seeds"][i]),
                                  predictor=predictor)
        while not req.done and time.perf_counter() - t0 < budget_s:
            req.step()
    return count[0], time.perf_counter() - t0


def cpu_measure(cfg_name, steps, budget_s, procs):
    import multiprocessing as mp
    ctx = mp.get_context("fork")
    with ctx.Pool(procs, initializer=_cpu_init, initargs=(cfg_name, 64, 4242)) as pool:
        pool.map(_cpu_run, [0.2] * procs)            # warm
        total_bs, total_t = 0, 0.0
        per_step = []
        for _ in range(steps):
            t0 = time.perf_counter()
            res = pool.map(_cpu_run, [budget_s] * procs)
            dt = time.perf_counter() - t0
            bs = sum(r[0] for r in res)
            total_bs += bs
            total_t += dt
            per_step.append(bs / dt)
    return total_bs / total_t, per_step


def cpu_baseline_entry(cfg_name, budget_total=12.0):
    procs = os.cpu_count() or 1
    steps = 3
    val, _ = cpu_measure(cfg_name, steps, budget_total / steps, procs)
    cfg = CONFIGS[cfg_name]
    return {"value": val, "unit": UNIT, "cores": procs, "kind": "port",
            "sample": f"oracle/port.py DuchessRun restatement + numpy pooled LN probe "
                      f"(T={cfg['T']}, H={cfg['H']}, L={cfg['L']}) on {cfg['preset']} requests "
                      f"(c={cfg['c']}), each branch-step scoring the next of a 64 MiB pool of "
                      f"distinct windows per process, {procs} processes x {steps} x "
                      f"{budget_total/steps:.1f} s"}


def cpu_fork_or_train(args):
    """CPU references for C4 (serial CoW restatement) and C5 (numpy fp32 BLAS
    gradient on all threads), each step a bounded sample."""
    from oracle import extensions as ext
    procs = os.cpu_count() or 1
    if args.config == "c4":
        R, roots, nf, bt, kvb = 24, 16, 48, 16, 4096
        pos, forks = make_fork_trace(R, roots, nf, bt, 256, seed=31)
        rows_per = roots + nf
        nblk = -(-pos // bt)
        table = np.full((R * rows_per, 256), -1, dtype=np.int32)
        nxt = 0
        for r in range(R):
            for b in range(roots):
                table[r * rows_per + b, :nblk[r, b]] = np.arange(nxt, nxt + nblk[r, b])
                nxt += nblk[r, b]
        n_blocks = nxt + R * nf
        ref = np.ones(n_blocks, dtype=np.int32)
        free = np.arange(nxt, n_blocks, dtype=np.int32)
        kv = np.zeros(n_blocks * bt * kvb, dtype=np.uint8)
        times = []
        for _ in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            ext.cow_fork_ref(forks, None, table, ref, free, 0, kv, kvb, bt, rows_per)
            times.append(time.perf_counter() - t0)
        dt = sum(times[args.warmup:])
        val, unit, sample = R * nf * args.steps / dt, "forks/s", \
            f"oracle/extensions.cow_fork_ref over {R} requests x {nf} forks, 1 core"
        cores = 1
    else:
        H, n = 8192, 65536
        rng = np.random.default_rng(0)
        X = rng.standard_normal((n, H), dtype=np.float32)
        y = (rng.random(n) < 0.5).astype(np.float32)
        w = (rng.standard_normal(H + 1) / 90).astype(np.float32)
        times = []
        for _ in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            z = X @ w[:-1] + w[-1]
            r = 1.0 / (1.0 + np.exp(-z)) - y
            _g = np.concatenate([X.T @ r, [r.sum()]]) / n
            times.append(time.perf_counter() - t0)
        dt = sum(times[args.warmup:])
        val, unit, sample = n * args.steps / dt, "rows/s", \
            f"numpy fp32 BLAS gradient on {n} x {H} rows, all threads"
        cores = procs
    return {"impl": "reference", "metric": f"{args.config} CPU reference", "value": val,
            "unit": unit, "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int32" if args.config == "c4" else "f32",
            "data": "synthetic", "config": {"workload": args.config.upper() + " (CPU)"},
            "cpu_baseline": {"value": val, "unit": unit, "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": val, "unit": unit, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def cpu_c3tc(n=4096, reps=3):
    """CPU reference for the C3 tensor-core MLP probe: the reference's
    mlp_forward (predictor.py:126-151; LN -> 5120x2048 ReLU -> 1 logit) as
    numpy fp32 BLAS on all threads over a bounded sample of windows."""
    K, NH = 5120, 2048
    rng = np.random.default_rng(0)
    X = rng.standard_normal((n, K), dtype=np.float32)
    W1 = (rng.standard_normal((K, NH)) / np.sqrt(K)).astype(np.float32)
    b1 = np.zeros(NH, dtype=np.float32)
    w2 = (rng.standard_normal(NH) / np.sqrt(NH)).astype(np.float32)
    g = rng.uniform(0.5, 1.5, K).astype(np.float32)
    beta = rng.uniform(-0.1, 0.1, K).astype(np.float32)
    times = []
    for _ in range(reps + 1):
        t0 = time.perf_counter()
        mu = X.mean(axis=1, keepdims=True)
        var = X.var(axis=1, keepdims=True)
        z = (X - mu) / np.sqrt(var + 1e-5) * g + beta
        h = np.maximum(z @ W1 + b1, 0.0)
        _logit = h @ w2
        times.append(time.perf_counter() - t0)
    dt = sum(times[1:])
    return {"value": n * reps / dt, "unit": "branch-steps/s", "cores": os.cpu_count() or 1,
            "kind": "port", "sample": f"numpy fp32 BLAS mlp_forward (LN, {K}->{NH} ReLU, head) "
                                      f"over {n} windows x {reps}, all threads"}


def run_reference(args, cfg):
    if args.config in ("difficulty", "sim", "baselines", "c3tc"):
        cb = {"difficulty": cpu_difficulty, "sim": cpu_sim, "baselines": cpu_baselines,
              "c3tc": cpu_c3tc}[args.config]()
        return {"impl": "reference", "metric": f"{args.config} CPU reference", "value": cb["value"],
                "unit": cb["unit"], "n_gpus": args.gpus, "steps": 1, "warmup": 0,
                "ms_per_step": None, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32" if args.config == "c3tc" else "f64",
                "data": "synthetic",
                "config": {"workload": args.config + " (CPU)"}, "cpu_baseline": cb,
                "e2e": {"value": cb["value"], "unit": cb["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
    if cfg is None:
        return cpu_fork_or_train(args)
    procs = os.cpu_count() or 1
    total = args.steps + args.warmup
    budget = max(0.5, min(5.0, 120.0 / max(total, 1)))
    import multiprocessing as mp
    ctx = mp.get_context("fork")
    with ctx.Pool(procs, initializer=_cpu_init, initargs=(args.config, 64, 4242)) as pool:
        for _ in range(args.warmup):
            pool.map(_cpu_run, [budget] * procs)
        total_bs, total_t = 0, 0.0
        for _ in range(args.steps):
            t0 = time.perf_counter()
            res = pool.map(_cpu_run, [budget] * procs)
            total_t += time.perf_counter() - t0
            total_bs += sum(r[0] for r in res)
    val = total_bs / total_t
    return {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_t / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": f"{args.config.upper()} (CPU port)",
                                        "requests": cfg["R"], "branches": cfg["c"],
                                        "hidden": cfg["H"], "layers": cfg["L"],
                                        "window": cfg["T"]},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": procs, "kind": "port",
                         "sample": f"{procs} processes x {budget:.2f} s per step of "
                                   f"oracle/port.py DuchessRun + numpy pooled probe, each "
                                   f"branch-step scoring the next of a 64 MiB pool of distinct "
                                   f"windows per process (streamed from DRAM like the GPU arm)"},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2",
                    choices=sorted(CONFIGS) + ["c3tc", "c4", "c5", "difficulty", "sim",
                                               "baselines"])
    ap.add_argument("--k1", default="list", choices=["list", "mask", "ldg"],
                    help="K1 variant: persistent TMA over the compacted survivor list "
                         "(default), TMA over the row mask, or the per-window LDG kernel")
    ap.add_argument("--mode", default="split", choices=["fused", "split"],
                    help="split (default): K1 launch + duchess_round launch per round; "
                         "fused: one duchess_step launch per round (see DESIGN.md 7)")
    ap.add_argument("--shards", type=int, default=None,
                    help="independent request shards (engines on separate CUDA streams) per "
                         "GPU; default 2 for c2 / c3, 1 otherwise")
    ap.add_argument("--shard-order", default=None, choices=["turns", "overlap"],
                    help="turns: the shards' scorers take turns (event chain); overlap: they "
                         "run concurrently (default overlap for c2, turns for c3)")
    ap.add_argument("--graph", action="store_true",
                    help="replay the round loop as a CUDA graph (one slab rotation per graph)")
    ap.add_argument("--k1-every", type=int, default=8,
                    help="bracket K1 with CUDA events on every N-th timed step")
    ap.add_argument("--nsplit", type=int, default=2)
    ap.add_argument("--threads", type=int, default=128)
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    cfg = CONFIGS.get(args.config)
    if args.shards is None:
        # two request shards per GPU on two streams hide each shard's round
        # kernel under the other's scoring
        args.shards = 2 if args.config in ("c2", "c3", "c3t1") else 1
    if args.shard_order is None:
        # concurrent scorers also fill each other's launch ramp and tail
        # (C3 with two-row stages: 5.64 vs 5.48-5.52 M/s taking turns)
        args.shard_order = "overlap" if args.config in ("c2", "c3", "c3t1") else "turns"
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args, cfg)), flush=True)
        return
    if world > 1:
        import torch
        # DUCHESS_BENCH_BACKEND=gloo (test only): exercise the multi-rank path on
        # a box with fewer GPUs than ranks (ranks share GPUs round-robin)
        backend = os.environ.get("DUCHESS_BENCH_BACKEND", "nccl")
        if backend != "nccl":
            local_rank %= torch.cuda.device_count()
        torch.cuda.set_device(local_rank)
        torch.distributed.init_process_group(backend)
    if args.config == "c4":
        out = run_fork_bench(args, rank, world, local_rank)
    elif args.config == "c5":
        out = run_train_bench(args, rank, world, local_rank)
    elif args.config == "c3tc":
        out = run_tc_bench(args, rank, world, local_rank)
    elif args.config == "difficulty":
        out = run_difficulty_bench(args, rank, world, local_rank)
    elif args.config == "sim":
        out = run_sim_bench(args, rank, world, local_rank)
    elif args.config == "baselines":
        out = run_baselines_bench(args, rank, world, local_rank)
    elif args.mode == "split" and args.k1 == "list" and not args.graph and args.shards > 1:
        out = run_gpu_sharded(args, cfg, rank, world, local_rank)
    else:
        out = run_gpu(args, cfg, rank, world, local_rank)
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline and cfg is not None:
            out["cpu_baseline"] = cpu_baseline_entry(args.config)
        elif world == 1 and not args.no_cpu_baseline and args.config in ("c4", "c5"):
            import copy
            small = copy.copy(args)
            small.steps, small.warmup = 3, 1           # bounded CPU sample
            out["cpu_baseline"] = cpu_fork_or_train(small)["cpu_baseline"]
        elif world == 1 and not args.no_cpu_baseline and args.config == "c3tc":
            out["cpu_baseline"] = cpu_c3tc()
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
