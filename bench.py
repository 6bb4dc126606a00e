"""Benchmark: branch-steps/s scored + decided (DUCHESS probe + orchestration).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2|c1|c3|c3t1|c4|c5|c3tc|baselines|difficulty|sim]

One step = one orchestration round over every request slot on the GPU:
duchess_score_active (K1: pooled LayerNorm + linear probe over each
survivor's activation window, read from HBM) -> duchess_round (K2: decide the
round: predict / early-terminate / branch-out / request termination + vote,
then refill and advance every slot into the next round) -> duchess_kv_round
(K3: the round's branch-outs share their root's paged KV blocks copy-on-write,
ended branches release theirs, decoding branches grow; launched overlapped
with the next round's K1). A branch-step is one survivor scored and decided
(one `self._predict` call in reference orchestrator.py:358-362).

Default workload at N = 1 (BASELINE.json configs[1], "C2"): 256 request
slots x 16 branch slots, hidden 4096, bf16 activations, 32-token pooling
window, one probe layer, math-like knobs with max_branches=16
(presets.py:55-59), a cycling pool of 2048 synthetic requests (64 templates
each) admitted in easiest-first order, a paged KV cache of 16-token blocks
with 4096 B of KV per token (one Llama-3-8B layer slice; `--config c2nokv`
drops it). Activations: rotating buffers per
shard (> the 126 MB L2, so every step streams from HBM). The slots are split
into two independent request shards stepping on two CUDA streams
(serving.ShardedEngine: requests never interact), so each shard's
latency-bound round kernel runs while the other shard's scorer streams.

Under torchrun (N > 1) the default stays C2, weak-scaled: every rank serves
one GPU's C2 workload (256 slots) from its own share of a pool N times as large,
so value = the whole job's branch-steps / the max-over-ranks time ("scaling":
"weak"). `--config c3` (and c3t1 / c3mlp) strong-scales BASELINE configs[2]:
its 1024 request slots and pool are split over the ranks. No data-path
collective either way (requests are independent); barrier + max-over-ranks
timing.

--impl reference times the reference's own DuchessRun + mlp_forward (vendored
unmodified into oracle/_ref by oracle/vendor_ref.py; the restatement
oracle/port.py when absent) with a predictor= that pools each distinct window
(fp64 mean over T) on all host cores.
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
    # C2 (configs[1]) with K3 in the round: a paged KV cache (16-token blocks, one
    # Llama-3-8B layer slice of KV = 2*8*128*2 = 4096 B per token) forked / grown /
    # released every round, so one step = K1 + K2 + K3 (north_star's three kernels)
    "c2": dict(R=256, c=16, L=1, T=32, H=4096, dtype="bf16", preset="math-like", pool=2048,
               kv=4096),
    # the same step without the KV cache (K1 + K2 only; the round-1 default)
    "c2nokv": dict(R=256, c=16, L=1, T=32, H=4096, dtype="bf16", preset="math-like",
                   pool=2048),
    "c1": dict(R=8, c=8, L=1, T=1, H=4096, dtype="f32", preset="gsm8k-like", pool=128),
    "c3": dict(R=1024, c=32, L=4, T=32, H=5120, dtype="bf16", preset="math-like", pool=4096),
    # C3 with the paper's correctness probe per layer (LN -> 2048 ReLU -> 1024 ReLU ->
    # 1) on the tensor cores: 4 probe layers batched, last token
    "c3mlp": dict(R=1024, c=32, L=4, T=1, H=5120, dtype="bf16", preset="math-like", pool=4096,
                  mlp=(2048, 1024)),
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


def k3_write_bytes():
    """DRAM bytes written by one fork_exec launch (committed ncu capture)."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "k3_traffic.json")))
    if not files:
        return None
    with open(files[-1]) as f:
        return json.load(f).get("dram_write_bytes")


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


def load_tc_peaks():
    """(sustained, burst) measured dense bf16 TFLOP/s (MEASURED_PEAKS.json),
    else the B200_PROFILING.md fallbacks."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["bf16_tflops_sustained"]), float(p["bf16_tflops"]), "measured"
    except Exception:  # noqa: BLE001
        return 1349.2, 1650.0, "fallback"


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


def make_mlp_probe(H, L, hidden, seed=0):
    """L random-init probes of the paper's architecture: LN affine,
    He-scaled ReLU layers, a small head. Returns per layer (weights, biases,
    ln_gain, ln_bias) as float64 arrays (MlpWeights layout, matrices (out, in))."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(L):
        dims = [H, *hidden, 1]
        ws = [rng.normal(0.0, np.sqrt(2.0 / dims[k]), (dims[k + 1], dims[k]))
              for k in range(len(dims) - 1)]
        ws[-1] *= 0.5
        bs = [rng.normal(0.0, 0.05, dims[k + 1]) for k in range(len(dims) - 1)]
        out.append((ws, bs, rng.uniform(0.5, 1.5, H), rng.uniform(-0.1, 0.1, H)))
    return out


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
def measure_read_peak(dev, buf=None, reps=6):
    """Read-only HBM ceiling on this GPU, measured live: best of `reps`
    passes of duchess_read_stream over >= 4 GiB (CUDA events)."""
    import torch

    from paper_2509_24957_b200 import _lib
    lib = _lib.load()
    own = buf is None or buf.numel() * buf.element_size() < (4 << 30)
    if own:
        buf = torch.empty(4 << 30, dtype=torch.uint8, device=dev)
        buf.fill_(1)
    nbytes = buf.numel() * buf.element_size() // 16 * 16
    sink = torch.zeros(4, dtype=torch.int32, device=dev)
    st = torch.cuda.current_stream(dev)
    best = None
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        _lib.check(lib.duchess_read_stream(buf.data_ptr(), nbytes, sink.data_ptr(),
                                           st.cuda_stream), "duchess_read_stream")
        b.record(st)
        b.synchronize()
        gbs = nbytes / (a.elapsed_time(b) / 1e3) / 1e9
        best = gbs if best is None else max(best, gbs)
    del buf
    return best


def measure_write_peak(dev, reps=6):
    """Write-only HBM ceiling on this GPU, measured live: best of `reps`
    passes of duchess_write_stream (16-byte streaming stores) over 4 GiB."""
    import torch

    from paper_2509_24957_b200 import _lib
    lib = _lib.load()
    buf = torch.empty(4 << 30, dtype=torch.uint8, device=dev)
    nbytes = buf.numel()
    st = torch.cuda.current_stream(dev)
    best = None
    for r in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        _lib.check(lib.duchess_write_stream(buf.data_ptr(), nbytes, r, st.cuda_stream),
                   "duchess_write_stream")
        b.record(st)
        b.synchronize()
        gbs = nbytes / (a.elapsed_time(b) / 1e3) / 1e9
        best = gbs if best is None else max(best, gbs)
    del buf
    return best


DATASHEET_HBM_GBS = 8000.0   # B200 HBM3e datasheet figure


def roofline_figures(achieved, read_peak):
    """The achieved GB/s against the three denominators BASELINE.md 2 asks
    for: the driver's measured copy peak (the line's `peak`), the 8 TB/s
    datasheet figure and the read-only stream measured in this run."""
    peak, kind = load_peaks()
    return {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "peak_kind": kind, "peak_note": PEAK_NOTE,
            "vs_datasheet": {"peak": DATASHEET_HBM_GBS, "frac": achieved / DATASHEET_HBM_GBS},
            "vs_read_stream": (None if read_peak is None else
                               {"peak": read_peak, "frac": achieved / read_peak,
                                "how": "duchess_read_stream (read-only persistent kernel, "
                                       ">= 4 GiB, best of 6, CUDA events) measured in this run"})}


GATE_STEPS = 24      # timed steps enqueued before the gate opens


class Gate:
    """duchess_gate on a stream: the GPU holds it until release() (a store to
    pinned host memory) or a 10 s timeout, so a timed region can be enqueued
    before it starts. check() raises if the gate timed out (the host did not
    release it: the timing would then include host time). Disabled with
    --no-gate (under a profiler, which serialises launches)."""

    def __init__(self, dev, enabled=True):
        import torch
        self.enabled = enabled
        self.flag = torch.zeros(1, dtype=torch.int32).pin_memory()
        self.timed_out = torch.zeros(1, dtype=torch.int32, device=dev)

    def hold(self, stream):
        if not self.enabled:
            return
        from paper_2509_24957_b200 import _lib
        lib = _lib.load()
        _lib.check(lib.duchess_gate(self.flag.data_ptr(), 10_000_000_000,
                                    self.timed_out.data_ptr(), stream.cuda_stream), "duchess_gate")

    def release(self):
        self.flag.fill_(1)

    def check(self) -> bool:
        """True when the gate opened by release(); False when it gave up on its
        timeout (the timed region then includes host enqueue time, reported in
        the line's config as gate_timed_out)."""
        if self.enabled and int(self.timed_out.item()):
            print("warning: launch gate timed out; the timed region includes host time",
                  file=sys.stderr)
            return False
        return True


# Configs whose N > 1 run splits the config's requests over the ranks (BASELINE
# configs[2]: "1024 requests ... sharded over 2/4/8 B200"); the others keep the
# per-GPU workload fixed and add GPUs (weak scaling).
STRONG_SCALED = ("c3", "c3t1", "c3mlp")


def serving_plan(cfg_name, world, rank):
    """Slots of this rank, its share of the request pool, and the pool size to
    generate. N = 1: the config as BASELINE.json states it. N > 1, C3 variants:
    strong scaling — the config's R request slots and its pool are split over
    the ranks (shard_range, contiguous). N > 1, others (C1 / C2: one GPU's
    workload): weak scaling — every rank serves R slots from its own share of a
    pool N times as large. No data-path collective either way (requests are
    independent)."""
    from paper_2509_24957_b200.distributed import shard_range
    cfg = CONFIGS[cfg_name]
    if cfg_name in STRONG_SCALED or world == 1:
        lo, hi = shard_range(cfg["R"], rank, world)
        return hi - lo, shard_range(cfg["pool"], rank, world), cfg["pool"]
    pool = cfg["pool"] * world
    return cfg["R"], shard_range(pool, rank, world), pool


def run_serving(args, cfg, rank, world, local_rank):
    """C1/C2/C3/C3-T1: the serving loop (serving.ShardedEngine): per round and
    request shard, duchess_score_active (K1) + duchess_round (K2)."""
    import torch

    from paper_2509_24957_b200 import _lib
    from paper_2509_24957_b200.engine import pack_pool
    from paper_2509_24957_b200.probe import ProbeBank, fill_windows
    from paper_2509_24957_b200.scheduler import difficulty_queue
    from paper_2509_24957_b200.serving import ShardedEngine

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    S = args.shards
    L, T, H, C = cfg["L"], cfg["T"], cfg["H"], cfg["c"]
    R, (plo, phi), pool = serving_plan(args.config, world, rank)
    if R % S:
        raise SystemExit(f"--shards {S} must divide this rank's {R} request slots")
    tdtype = torch.bfloat16 if cfg["dtype"] == "bf16" else torch.float32
    esz = 2 if cfg["dtype"] == "bf16" else 4
    traces, knobs, seeds = make_workload(dict(cfg, pool=pool), seed=1000)   # same on every rank
    order = difficulty_queue([t.difficulty for t in traces], device=dev)
    queue = [p for p in order if plo <= p < phi]               # this rank's share, easiest first
    if cfg.get("mlp"):
        from paper_2509_24957_b200.mlp_probe import MlpProbeBank
        from paper_2509_24957_b200.predictor import MlpWeights
        hid = list(cfg["mlp"])
        bank = MlpProbeBank([MlpWeights(H, hid, 1, ["relu"] * len(hid), ws, bs, g, beta)
                             for ws, bs, g, beta in make_mlp_probe(H, L, hid)], device=dev)
    else:
        w, b, g, beta = make_probe(H, L)
        bank = ProbeBank.from_linear(w, b, g, beta, device=dev)
    rows = (R // S) * C
    slab_bytes = rows * L * T * H * esz
    n_slabs = 4 if slab_bytes * S < (256 << 20) else max(2, min(4, int((4 << 30) // (slab_bytes * S)) or 2))
    packed = pack_pool(traces, seeds, dev)
    kv = (dict(block_tokens=16, kv_bytes_per_token=cfg["kv"]) if cfg.get("kv") else None)
    srv = ShardedEngine(traces, knobs, seeds, bank, n_slots=R, shards=S, queue=queue, cycle=True,
                        T=T, dtype=tdtype, device=dev, n_buffers=n_slabs, packed=packed, kv=kv)
    for k, sh in enumerate(srv.shards):
        for i, a in enumerate(sh["acts"]):
            fill_windows(a, 7000 + 31 * rank + 7 * k + i)
    read_peak = measure_read_peak(dev, srv.shards[0]["acts"][0]) if rank == 0 else None
    main = torch.cuda.current_stream(dev)

    srv.begin()
    for i in range(BURN_IN_ROUNDS + args.warmup):
        srv.step(i)
    srv.join()
    torch.cuda.synchronize(dev)
    first = BURN_IN_ROUNDS + args.warmup
    graph = None
    if args.graph:
        # one CUDA graph = one rotation of the activation buffers (n_slabs
        # rounds of every shard, the shard streams forked / joined inside),
        # replayed: removes the host launch cost that bounds small configs
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            srv.fork()
            for j in range(n_slabs):
                srv.step(first + j)
            srv.join()
        args.steps = -(-args.steps // n_slabs) * n_slabs
        graph.replay()                  # one rotation untimed
        torch.cuda.synchronize(dev)
    c0 = srv.counters()
    kv0 = srv.kv_counters()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    clocks = ClockSampler(local_rank) if rank == 0 else None
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # The timed steps are enqueued behind a gate kernel (released once the first
    # GATE_STEPS steps are queued), so the device time measures the steps
    # back to back rather than the host's first launches (nvbench's blocking
    # kernel); the barrier + synchronize bracket is unchanged. Every kernel of
    # a step ran in the warm-up, so no lazy module load (which would wait for
    # the gate) happens while it holds.
    gate = Gate(dev, enabled=not args.no_gate)
    gate.hold(main)
    ev0.record(main)
    if graph is not None:
        for r in range(args.steps // n_slabs):
            graph.replay()
            if (r + 1) * n_slabs >= GATE_STEPS:
                gate.release()
    else:
        srv.fork()
        for i in range(args.steps):
            srv.step(first + i, timed=(S == 1 and i % args.k1_every == 0))
            if i + 1 == GATE_STEPS:
                gate.release()
        srv.join()
    ev1.record(main)
    gate.release()
    torch.cuda.synchronize(dev)
    gate_ok = gate.check()
    clk = clocks.stop() if clocks else None
    cnt = srv.counters() - c0
    kv1 = srv.kv_counters()
    ms = ev0.elapsed_time(ev1)
    if S == 1 and graph is not None:
        # events inside a replayed graph are not meaningful: K1 is timed in an
        # eager pass right after the timed region (same state and shapes)
        srv.fork()
        for i in range(8 * args.k1_every):
            srv.step(i, timed=(i % args.k1_every == 0))
        srv.join()
        torch.cuda.synchronize(dev)
    if world > 1:
        torch.distributed.barrier()
    branch_steps = int(cnt[_lib.CNT_BRANCH_STEPS])
    stats = torch.tensor([ms, float(branch_steps)], dtype=torch.float64, device=dev)
    if world > 1:
        tmax = stats[:1].clone()
        torch.distributed.all_reduce(tmax, op=torch.distributed.ReduceOp.MAX)
        tot = stats[1:2].clone()
        torch.distributed.all_reduce(tot, op=torch.distributed.ReduceOp.SUM)
        ms_all, bs_all = float(tmax[0]), float(tot[0])
    else:
        ms_all, bs_all = ms, float(branch_steps)

    e2e = run_serving_e2e(args, srv, rows, L, T, H, tdtype, dev, world)
    if rank != 0:
        return None
    bytes_per_bs = T * H * esz * L
    step_s = ms / args.steps / 1e3
    k1_us = [a.elapsed_time(b) * 1e3 for a, b in srv.scorer_events()]
    k1_avg_s = sum(k1_us) / max(len(k1_us), 1) / 1e6
    bytes_per_launch = branch_steps / args.steps / S * bytes_per_bs
    if S > 1:
        # the shards' scorer launches run concurrently and share HBM: the
        # step's scoring bytes over the WHOLE step time (round kernels
        # included) is the conservative figure
        achieved = bytes_per_launch * S / step_s / 1e9
        kernel = (f"duchess_score_active (K1{', score_rows_kernel' if T == 1 else ''}): the "
                  f"{S} shards' concurrent launches, scoring bytes per step / whole step time")
    else:
        achieved = bytes_per_launch / k1_avg_s / 1e9
        kernel = (f"duchess_score_active (K1{', score_rows_kernel' if T == 1 else ''}) per "
                  f"launch (CUDA events on the shard stream)")
    roof = roofline_figures(achieved, read_peak)
    ratio, src = k1_traffic_ratio(T)
    roof.update({"kernel": kernel, "bytes_per_launch": bytes_per_launch,
                 "bytes_per_branch_step": bytes_per_bs,
                 "k1_us_per_launch": k1_avg_s * 1e6 if k1_us else None,
                 "k1_launches_timed": len(k1_us),
                 "traffic": None if ratio is None else ratio * bytes_per_launch,
                 "traffic_source": src})
    if cfg.get("mlp"):
        # tensor-core bound: algorithmic FLOPs of the survivors (the GEMMs run
        # dense over all R*C slots; the dense figure is reported beside it)
        flops_bs = bank.flops(1)
        fl_launch = branch_steps / args.steps / S * flops_bs
        dense = rows * flops_bs
        t_s = k1_avg_s if k1_us else step_s
        sus, burst, _kind = load_tc_peaks()
        tfl = fl_launch / t_s / 1e12
        roof = {"bound": "tensor", "achieved": tfl, "peak": sus, "unit": "TFLOP/s",
                "frac": tfl / sus if sus else None, "traffic": None,
                "peak_kind": "measured bf16 dense, sustained (MEASURED_PEAKS.json); the "
                             "scorer runs back to back inside a long step",
                "vs_burst": {"peak": burst, "frac": tfl / burst if burst else None},
                "dense_tflops": dense / t_s / 1e12,
                "kernel": "MlpProbeBank: duchess_tc_linear_grouped (LN fold + ReLU, 4 layers) + "
                          "duchess_mlp_probe_tc_grouped (ReLU + head), events around both",
                "flops_per_branch_step": flops_bs, "flops_per_launch": fl_launch,
                "dense_flops_per_launch": dense,
                "scorer_us_per_launch": t_s * 1e6, "launches_timed": len(k1_us)}
    strong = world > 1 and args.config in STRONG_SCALED
    weak_multi = world > 1 and not strong
    return {
        "metric": METRIC, "value": bs_all / (ms_all / 1e3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_all / args.steps,
        "higher_is_better": True, "scaling": "strong" if strong else "weak",
        "vs_baseline": None, "dtype": cfg["dtype"],
        "data": "synthetic (counter-hashed N(0,1) activations with outlier channels; "
                "generate_synthetic workload, random-init probe)",
        "config": {"workload": f"{args.config.upper()}: {cfg['R']} request slots x {C} branches"
                   f"{f' split over {world} GPUs ({R} per GPU)' if strong else ''}"
                   f"{f' on each of {world} GPUs' if weak_multi else ''}, hidden {H}, "
                   f"{L} probe layer(s){' (mean of probabilities)' if L > 1 else ''}, T={T} "
                   f"pooling window, {cfg['dtype']}, {cfg['preset']} knobs, cycling pool of "
                   f"{pool} requests (easiest-first{', split over the GPUs' if world > 1 else ''}), "
                   f"{n_slabs} rotating activation buffers per shard "
                   f"({slab_bytes * S / 2**30:.2f} GiB per rotation step, > L2); {S} request "
                   f"shard(s) per GPU on {S} CUDA stream(s)",
                   "requests": cfg["R"] * (world if weak_multi else 1), "branches": C,
                   "hidden": H, "layers": L, "window": T,
                   "pool": pool, "slots_per_gpu": R, "shards_per_gpu": S,
                   "launch": "CUDA graph replay" if graph is not None else "eager streams (PDL)",
                   "l2": "inputs larger than L2 (rotating buffers)",
                   "burn_in_rounds": BURN_IN_ROUNDS,
                   "timed_region": f"CUDA events on the main stream around K steps; the first "
                                   f"{GATE_STEPS} steps are enqueued behind a launch gate "
                                   f"(duchess_gate) before the GPU starts them",
                   **({} if gate_ok else {"gate_timed_out": True}),
                   "parallelism": f"request-sharded x{world} GPUs x{S} streams"},
        "branch_steps_per_step": bs_all / args.steps,
        "roofline": roof,
        "e2e": e2e,
        "gpu_launches": (3 if kv1 else 2) * S * args.steps,
        "clocks": clk,
        "counters": {"ambiguous_draws": int(cnt[_lib.CNT_AMBIGUOUS]),
                     "finished_requests": int(cnt[_lib.CNT_FINISHED]),
                     "forks": int(cnt[_lib.CNT_FORKS]),
                     # predictions within the probe's 1e-4 logit tolerance of tau:
                     # an fp64 probe could have decided these `p > tau` the other way
                     "near_tau_predictions": int(cnt[_lib.CNT_NEAR_TAU])},
        **({"kv_cache": kv_report(kv0, kv1, args.steps, srv, cfg)} if kv1 else {}),
    }


def kv_report(kv0, kv1, steps, srv, cfg):
    """K3-in-the-round figures over the timed steps (PagedKVCache counters)."""
    sh = srv.shards[0]["kv"]
    d = {k: kv1[k] - kv0[k] for k in ("blocks_allocated", "blocks_released", "tail_bytes",
                                       "overflow")}
    how = {"lead": "duchess_kv_round (kv_round_kernel: forks incl. tail copies, releases, "
                   "appends) right after every duchess_round, releasing the next round's "
                   "scorer, which streams beside it (DUCHESS_KV_LEAD + "
                   "DUCHESS_SCORE_NO_INPUT_WAIT)",
           "overlap": "duchess_kv_round after the next round's scorer, beside it "
                      "(DUCHESS_KV_OVERLAP)",
           "fused": "duchess_round_kv (the round kernel applies its K3 update) + "
                    "duchess_kv_copy_tails"}[srv.kv_mode]
    return {"kernels": how, "kv_mode": srv.kv_mode,
            "block_tokens": sh.block_tokens, "kv_bytes_per_token": sh.kv_bytes_per_token,
            "blocks_per_slot": sh.P,
            "pool_gib": sum(s["kv"].t["kv_pool"].numel() for s in srv.shards) / 2**30,
            "blocks_allocated_per_step": d["blocks_allocated"] / steps,
            "blocks_released_per_step": d["blocks_released"] / steps,
            "tail_bytes_per_step": d["tail_bytes"] / steps,
            "overflow": d["overflow"],
            "peak_blocks_per_slot": kv1["peak_blocks_per_slot"]}


def run_serving_e2e(args, srv, rows, L, T, H, tdtype, dev, world):
    """The same round through the public API with the activations in pinned
    HOST memory: per round and shard, upload_survivors (one kernel gathers
    exactly the survivors' windows over PCIe), K1 + round, and a D2H read of
    the round records and actions (the RoundReports). The host buffers hold
    the same counter-hashed windows as the device buffers (copied from them)."""
    import torch

    from paper_2509_24957_b200 import _lib
    steps = max(2, min(args.e2e_steps, args.steps))
    row_bytes = L * T * H * torch.tensor([], dtype=tdtype).element_size()
    srv.flush_kv()
    for sh in srv.shards:
        sh["host"] = torch.empty((rows, L, T, H), dtype=tdtype, pin_memory=True)
        sh["host"].copy_(sh["acts"][0])
        sh["dslab"] = torch.empty_like(sh["host"], device=dev)
        sh["rec_h"] = torch.empty(sh["eng"].t["round_rec"].numel(), dtype=torch.int32,
                                  pin_memory=True)
        sh["act_h"] = torch.empty(sh["eng"].t["actions"].numel(), dtype=torch.int32,
                                  pin_memory=True)
    torch.cuda.synchronize(dev)

    # input path per shard: "gather" = duchess_gather_active (SM reads of the
    # host mapping), "dma" = the survivor list read back with the round records,
    # then one DMA per run of consecutive rows (duchess_upload_rows); "mixed" =
    # shard 0 by DMA, the others by gather, side by side on the link
    mode = args.e2e_upload
    if mode == "auto":
        # DMA runs pay ~4 us of copy-engine setup per run: a win for big windows
        # (C2 256 KB: 0.20 vs 0.19 M/s; C3 1.3 MB: 41.6 vs 37.5 K/s), a loss for
        # last-token rows (C1 16 KB: 0.43 vs 0.71 M/s; C3-T1 40 KB: 0.92 vs 1.25 M/s)
        mode = "dma" if row_bytes >= (128 << 10) else "gather"
    dma = [mode == "dma" or (mode == "mixed" and k == 0) for k in range(len(srv.shards))]
    list_bytes = [0]

    def step():
        order = [k for k in range(len(srv.shards)) if not dma[k]] + \
                [k for k in range(len(srv.shards)) if dma[k]]
        for k in order:
            sh = srv.shards[k]
            with torch.cuda.stream(sh["stream"]):
                eng = sh["eng"]
                if dma[k]:
                    rws = eng.survivor_rows_host(sh["stream"])
                    list_bytes[0] += 4 * (8 + len(rws))
                    eng.upload_rows(sh["host"], sh["dslab"], rws)
                else:
                    eng.upload_survivors(sh["host"], sh["dslab"])
                sh["scorer"].score_active(sh["dslab"], sh["logit"],
                                          eng.probs.view(rows, L), eng)
                eng.round()
                if sh["kv"] is not None:
                    sh["kv"].round()
                sh["rec_h"].copy_(eng.t["round_rec"], non_blocking=True)
                sh["act_h"].copy_(eng.t["actions"], non_blocking=True)
        for sh in srv.shards:
            sh["stream"].synchronize()

    step()
    c0 = srv.counters()
    if world > 1:
        torch.distributed.barrier()
    list_bytes[0] = 0
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    dt = time.perf_counter() - t0
    bs = int((srv.counters() - c0)[_lib.CNT_BRANCH_STEPS])
    st = torch.tensor([dt, float(bs)], dtype=torch.float64, device=dev)
    if world > 1:
        a = st[:1].clone()
        torch.distributed.all_reduce(a, op=torch.distributed.ReduceOp.MAX)
        b = st[1:].clone()
        torch.distributed.all_reduce(b, op=torch.distributed.ReduceOp.SUM)
        dt, bs = float(a[0]), float(b[0])
    for sh in srv.shards:
        for k in ("host", "dslab"):
            sh.pop(k)
    return {"value": bs / dt, "unit": UNIT,
            "h2d_bytes_per_step": bs / steps / max(world, 1) * row_bytes,
            "h2d": {"gather": "survivor windows only (duchess_gather_active over each shard's "
                              "active list)",
                    "dma": "survivor windows only, one DMA per run of consecutive survivor "
                           "rows (duchess_upload_rows; list read back with the round records)",
                    "mixed": "survivor windows only: shard 0 by DMA runs (duchess_upload_rows), "
                             "the other shard by duchess_gather_active, side by side"}[mode]
                   + "; average per rank; host buffers hold the counter-hashed windows",
            "upload": mode,
            "d2h_bytes_per_step": sum((sh["rec_h"].numel() + sh["act_h"].numel()) * 4
                                      for sh in srv.shards) + list_bytes[0] / steps,
            "steps": steps, "timing": "host wall clock, streams synchronised each step"}


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
    del flush
    wpeak = measure_write_peak(dev) if rank == 0 else None
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
                         "traffic": k3_traffic()[0], "traffic_source": k3_traffic()[1],
                         # the launch is write-dominated (ncu: ~4.3x more DRAM bytes
                         # written than read): its DRAM writes per second against a
                         # write-only stream measured in this run
                         "writes_vs_write_stream": (None if k3_write_bytes() is None or wpeak is None else {
                             "write_stream_gbs": wpeak,
                             "dram_write_gbs": k3_write_bytes() / (k3_ms / 1e3) / 1e9,
                             "frac": k3_write_bytes() / (k3_ms / 1e3) / 1e9 / wpeak})},
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
           "gpu_launches": (len(dims) + 1) * args.steps, "clocks": clk}
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
    """C5: one full-batch logistic-regression step over BASELINE's 4 194 304
    rows x 8192 (bf16), the rows split over the N ranks (strong scaling:
    4M / N rows per GPU, 64 GiB at N = 1): K4 over the rank's shard, the
    NCCL all-reduce of the 8193-float gradient (timed separately with events
    on the same stream), SGD update."""
    import torch
    from paper_2509_24957_b200.distributed import allreduce_sum, shard_range
    from paper_2509_24957_b200.probe import fill_windows
    from paper_2509_24957_b200.train import LogisticProbeTrainer
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    H = 8192
    n_total = int(os.environ.get("DUCHESS_C5_ROWS", 4194304))
    lo, hi = shard_range(n_total, rank, world)
    n_local = hi - lo
    X = torch.empty((n_local, 1, 1, H), dtype=torch.bfloat16, device=dev)
    fill_windows(X, 5000 + rank)
    X = X.view(n_local, H)
    g = torch.Generator(device=dev).manual_seed(5)
    w_true = torch.randn(H, generator=g, device=dev) / np.sqrt(H)
    y = torch.empty(n_local, device=dev)
    for a in range(0, n_local, 65536):
        z = X[a:a + 65536].float() @ w_true
        y[a:a + 65536] = (torch.rand(z.shape[0], generator=g, device=dev)
                          < torch.sigmoid(z)).float()
    del z
    tr = LogisticProbeTrainer(H, device=dev, lr=0.5)
    stream = torch.cuda.current_stream(dev)
    read_peak = measure_read_peak(dev, X) if rank == 0 else None
    for _ in range(args.warmup):
        tr.step(X, y, n_total)
    torch.cuda.synchronize(dev)
    if world > 1:
        torch.distributed.barrier()
    clocks = ClockSampler(local_rank) if rank == 0 else None
    k4_ev, ar_ev = [], []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        a.record(stream)
        tr.local_grad(X, y, 1.0 / n_total)
        b.record(stream)
        allreduce_sum(tr.grad)
        c.record(stream)
        k4_ev.append((a, b))
        ar_ev.append((b, c))
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
    k4_ms = sum(a.elapsed_time(b) for a, b in k4_ev) / args.steps
    ar_us = sum(a.elapsed_time(b) for a, b in ar_ev) / args.steps * 1e3
    bytes_launch = n_local * (H * 2 + 4)
    achieved = bytes_launch / (k4_ms / 1e3) / 1e9
    roof = roofline_figures(achieved, read_peak)
    roof.update({"kernel": "duchess_lr_grad (K4)", "bytes_per_launch": bytes_launch,
                 "k4_us_per_launch": k4_ms * 1e3, "traffic": None})
    backend = torch.distributed.get_backend() if world > 1 else None
    return {"metric": "probe-training rows/s (C5 logistic regression, full-batch step)",
            "value": n_total / (ms / 1e3), "unit": "rows/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic N(0,1) activations, labels ~ Bernoulli(sigmoid(X w*))",
            "config": {"workload": f"C5: {n_total} rows x {H} bf16 split over {world} GPU(s) "
                                   f"({n_local} rows, {bytes_launch / 2**30:.1f} GiB on rank 0), "
                                   f"grad + all-reduce (8193 f32) + SGD",
                       "rows": n_total, "rows_per_gpu": n_local, "hidden": H},
            "roofline": roof,
            "allreduce": {"us_per_step": ar_us, "bytes": (H + 1) * 4,
                          "backend": backend or "none (one rank: no collective)"},
            "gpu_launches": 3 * args.steps, "clocks": clk}


# ---------------------------------------------------------------------------
# CPU reference — only here and in tests may oracle/ (incl. the vendored
# reference in oracle/_ref) run.

_CPU = {}
CPU_POOL_BYTES = 64 << 20      # activation windows per CPU process (16 processes: 1 GiB)


def cpu_kind() -> str:
    """'reference' when the unmodified reference is vendored in oracle/_ref
    (oracle/vendor_ref.py, checked against its SHA-256 manifest), else 'port'
    (the pinned restatement oracle/port.py)."""
    from oracle import vendor_ref
    if vendor_ref.available():
        ref = os.path.join(ROOT, "oracle", "_ref")
        if ref not in sys.path:
            sys.path.insert(0, ref)
        return "reference"
    return "port"


def _cpu_init(cfg_name, n_req, seed, kind):
    # one BLAS thread per process: variant 1 is one core, variant 2 one process
    # per core (a multi-threaded BLAS in each of 16 processes oversubscribes)
    try:
        from threadpoolctl import threadpool_limits
        _CPU["blas_limit"] = threadpool_limits(1)
    except Exception:  # noqa: BLE001
        pass
    cfg = CONFIGS[cfg_name]
    H, T, L = cfg["H"], cfg["T"], cfg["L"]
    w, b, g, beta = make_probe(H, L)
    if kind == "reference":
        # the reference itself: generate_synthetic, DuchessRun, mlp_forward
        from branchsim.orchestrator import DuchessRun, OrchestratorConfig
        from branchsim.predictor import MlpWeights, mlp_forward
        from branchsim.workload import SyntheticParams, generate_synthetic
        params = SyntheticParams(templates_per_request=64, **PRESET_GEN[cfg["preset"]])
        traces = generate_synthetic(params, n_req, seed=seed).requests
        knobs = OrchestratorConfig(max_branches=cfg["c"], **PRESET_KNOBS[cfg["preset"]])
        if cfg.get("mlp"):
            hid = list(cfg["mlp"])
            probes = [MlpWeights(input_dim=H, layer_dims=hid, head_dim=1,
                                 activations=["relu"] * len(hid), weights=ws, biases=bs,
                                 ln_gain=gg, ln_bias=bb)
                      for ws, bs, gg, bb in make_mlp_probe(H, L, hid)]
        else:
            probes = [MlpWeights(input_dim=H, layer_dims=[], head_dim=1, activations=[],
                                 weights=[w[l].reshape(1, H).copy()], biases=[np.array([b[l]])],
                                 ln_gain=g[l].copy(), ln_bias=beta[l].copy()) for l in range(L)]

        def score(l, m):
            return float(mlp_forward(probes[l], m)[1][0])

        def make_run(trace, rng, predictor):
            return DuchessRun(trace, knobs, rng, predictor=predictor)
    else:
        from oracle import port
        params = port.GenParams(templates_per_request=64, **PRESET_GEN[cfg["preset"]])
        traces = port.generate(params, n_req, seed)
        knobs = port.Knobs(max_branches=cfg["c"], **PRESET_KNOBS[cfg["preset"]])

        if cfg.get("mlp"):
            from types import SimpleNamespace
            hid = list(cfg["mlp"])
            mlps = [SimpleNamespace(input_dim=H, layer_dims=hid, head_dim=1,
                                    activations=["relu"] * len(hid), weights=ws, biases=bs,
                                    ln_gain=gg, ln_bias=bb, bn_mean=None)
                    for ws, bs, gg, bb in make_mlp_probe(H, L, hid)]

            def score(l, m):
                return float(port.mlp_forward(mlps[l], m)[1][0])
        else:
            def score(l, m):
                return port.pooled_linear_probe(m[None, :], w[l], b[l], g[l], beta[l])[1]

        def make_run(trace, rng, predictor):
            return port.DuchessRequest(trace, knobs, rng, predictor=predictor)
    master = random.Random(seed + 1)
    seeds = [master.getrandbits(64) for _ in traces]
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
    _CPU.update(traces=traces, seeds=seeds, score=score, make_run=make_run, windows=pool,
                L=L, next=0, cursor=0)


def _cpu_run(budget_s):
    """Serve requests with the (reference's) DuchessRun for budget_s seconds;
    predictor= pools the next window (fp64 mean over T, the north-star's
    pooling) and scores it with mlp_forward per layer (mean of the layers'
    probabilities, as the GPU's combine=1). Returns (branch-steps, seconds)."""
    st = _CPU
    count = [0]
    score, L = st["score"], st["L"]

    def predictor(_tmpl, _position, _rng):
        count[0] += 1
        win = st["windows"][st["cursor"] % len(st["windows"])]
        st["cursor"] += 1
        ps = [score(l, win[l].mean(axis=0, dtype=np.float64)) for l in range(L)]
        return ps[0] if L == 1 else sum(ps) / L

    t0 = time.perf_counter()
    while time.perf_counter() - t0 < budget_s:
        i = st["next"] % len(st["traces"])
        st["next"] += 1
        req = st["make_run"](st["traces"][i], random.Random(st["seeds"][i]), predictor)
        while not req.done and time.perf_counter() - t0 < budget_s:
            req.step()
    return count[0], time.perf_counter() - t0


def cpu_measure(cfg_name, steps, budget_s, procs, kind, warmup=1):
    """Variant 1 (procs = 1) / variant 2 (procs = all cores; requests are
    independent): branch-steps/s over `steps` timed rounds of
    `budget_s` seconds per process."""
    import multiprocessing as mp
    ctx = mp.get_context("fork")
    with ctx.Pool(procs, initializer=_cpu_init, initargs=(cfg_name, 64, 4242, kind)) as pool:
        for _ in range(warmup):
            pool.map(_cpu_run, [min(budget_s, 0.5)] * procs)
        total_bs, total_t = 0, 0.0
        for _ in range(steps):
            t0 = time.perf_counter()
            res = pool.map(_cpu_run, [budget_s] * procs)
            total_t += time.perf_counter() - t0
            total_bs += sum(r[0] for r in res)
    return total_bs / total_t, total_t


def cpu_vectorised(cfg_name, budget_s=3.0):
    """Variant 3: vectorised numpy fp32 restatement of the
    scoring (pool over T -> LayerNorm -> dot -> sigmoid) over batches of
    distinct windows, BLAS on all threads; scoring only, no decisions."""
    cfg = CONFIGS[cfg_name]
    H, T, L = cfg["H"], cfg["T"], cfg["L"]
    if cfg.get("mlp"):
        return cpu_vectorised_mlp(cfg, budget_s)
    w, b, g, beta = make_probe(H, L)
    wg = (w * g).astype(np.float32)
    c1 = (np.einsum("lh,lh->l", w, beta) + b).astype(np.float32)
    n = max(64, int((256 << 20) // (L * T * H * 4)))
    X = np.random.default_rng(0).standard_normal((n, L, T, H), dtype=np.float32)
    done, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < budget_s:
        m = X.mean(axis=2)                                   # [n, L, H]
        mu = m.mean(axis=2, keepdims=True)
        z = (m - mu) / np.sqrt(((m - mu) ** 2).mean(axis=2, keepdims=True) + 1e-5)
        logit = np.einsum("nlh,lh->nl", z, wg) + c1
        _p = 1.0 / (1.0 + np.exp(-logit))
        done += n
    return done / (time.perf_counter() - t0)


def cpu_vectorised_mlp(cfg, budget_s=3.0):
    """Variant 3 for the MLP probe: numpy fp32, BLAS on all threads, batches of
    last-token windows through LN -> ReLU layers -> head per probe layer."""
    H, L = cfg["H"], cfg["L"]
    hid = list(cfg["mlp"])
    probes = make_mlp_probe(H, L, hid)
    prm = [([w.astype(np.float32) for w in ws], [bb.astype(np.float32) for bb in bs],
            g.astype(np.float32), beta.astype(np.float32)) for ws, bs, g, beta in probes]
    n = 512
    X = np.random.default_rng(0).standard_normal((n, L, H), dtype=np.float32)
    done, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < budget_s:
        for l, (ws, bs, g, beta) in enumerate(prm):
            x = X[:, l, :]
            mu = x.mean(axis=1, keepdims=True)
            z = (x - mu) / np.sqrt(((x - mu) ** 2).mean(axis=1, keepdims=True) + 1e-5) * g + beta
            for k in range(len(hid)):
                z = np.maximum(z @ ws[k].T + bs[k], 0.0)
            _p = 1.0 / (1.0 + np.exp(-(z @ ws[-1].T + bs[-1])))
        done += n
    return done / (time.perf_counter() - t0)


def host_info():
    import platform
    model = None
    try:
        out = os.popen("lscpu 2>/dev/null").read()
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
    except Exception:  # noqa: BLE001
        pass
    blas = None
    try:
        from threadpoolctl import threadpool_info
        blas = [{"api": d.get("internal_api"), "threads": d.get("num_threads")}
                for d in threadpool_info()]
    except Exception:  # noqa: BLE001
        pass
    return {"cpu_model": model, "os_cpu_count": os.cpu_count(),
            "python": platform.python_version(), "numpy": np.__version__, "blas": blas}


def cpu_baseline_entry(cfg_name, budget_total=12.0):
    """The GPU line's cpu_baseline: variant 2 (the reference on every host
    core) as `value`, variants 1 and 3 beside it, host description."""
    procs = os.cpu_count() or 1
    kind = cpu_kind()
    steps = 3
    v2, _ = cpu_measure(cfg_name, steps, budget_total / steps, procs, kind)
    v1, _ = cpu_measure(cfg_name, 1, 4.0, 1, kind)
    v3 = cpu_vectorised(cfg_name)
    cfg = CONFIGS[cfg_name]
    what = ("the unmodified reference (oracle/_ref/branchsim: generate_synthetic, DuchessRun, "
            "mlp_forward)" if kind == "reference" else "oracle/port.py (restatement)")
    return {"value": v2, "unit": UNIT, "cores": procs, "kind": kind,
            "sample": f"{what} with predictor= pooling (fp64 mean over T) + scoring each "
                      f"branch-step's next window of a 64 MiB pool of distinct windows "
                      f"(T={cfg['T']}, H={cfg['H']}, L={cfg['L']}), {cfg['preset']} requests "
                      f"(c={cfg['c']}), {procs} processes x {steps} x {budget_total/steps:.1f} s",
            "variants": {"1_one_core": {"value": v1, "cores": 1, "kind": kind},
                         "2_all_cores": {"value": v2, "cores": procs, "kind": kind},
                         "3_numpy_fp32_vectorised_scoring_only": {
                             "value": v3, "cores": procs, "kind": "port",
                             "note": "pool + LN + dot + sigmoid, numpy/BLAS all threads, "
                                     "no decisions"}},
            "host": host_info()}


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
    kind = cpu_kind()
    total = args.steps + args.warmup
    budget = max(0.5, min(5.0, 120.0 / max(total, 1)))
    val, total_t = cpu_measure(args.config, args.steps, budget, procs, kind, warmup=args.warmup)
    what = ("the unmodified reference (oracle/_ref/branchsim DuchessRun + mlp_forward)"
            if kind == "reference" else "oracle/port.py DuchessRun restatement + pooled probe")
    return {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_t / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": f"{args.config.upper()} (CPU {kind})",
                                        "requests": cfg["R"], "branches": cfg["c"],
                                        "hidden": cfg["H"], "layers": cfg["L"],
                                        "window": cfg["T"]},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": procs, "kind": kind,
                         "sample": f"{procs} processes x {budget:.2f} s per step of {what}, "
                                   f"predictor= pooling (fp64 mean over T) + scoring each "
                                   f"branch-step's next window of a 64 MiB pool of distinct "
                                   f"windows per process (streamed from DRAM like the GPU arm)",
                         "host": host_info()},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


# BASELINE configs measured after the C2 headline on the plain `python bench.py`
# run (N = 1), so every config's number comes from the driver's own run:
# configs[0] (c1), configs[2] per GPU (c3, its T = 1 row c3t1, its tensor-core
# MLP-probe variant c3mlp), configs[3] (c4), configs[4] per GPU (c5), and the
# the difficulty classifier, the baseline policies and
# run_simulation.
SECONDARY = ["c1", "c3", "c3t1", "c3mlp", "c4", "c5", "difficulty", "baselines", "sim"]
SECONDARY_TIMEOUT_S = 300
SECONDARY_KEYS = ("metric", "value", "unit", "ms_per_step", "steps", "warmup", "dtype",
                  "scaling", "config", "roofline", "e2e", "cpu_baseline", "clocks",
                  "gpu_launches", "counters", "error")


def run_secondary(names):
    """One `bench.py --config <name>` subprocess per name (same interpreter,
    default K / W, bounded by SECONDARY_TIMEOUT_S); returns {name: its JSON
    line, trimmed to the contract's keys} or {name: {"error": ...}}."""
    import subprocess
    res = {}
    for name in names:
        cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", name,
               "--secondary", "none"]
        if name in ("c3t1", "c3mlp"):
            # C3's own line carries the CPU baseline of this workload
            cmd += ["--e2e-steps", "4", "--no-cpu-baseline"]
        t0 = time.time()
        try:
            p = subprocess.run(cmd, capture_output=True, text=True, timeout=SECONDARY_TIMEOUT_S,
                               cwd=ROOT)
            lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
            if p.returncode != 0 or not lines:
                res[name] = {"error": f"rc={p.returncode}: {p.stderr.strip()[-300:]}"}
            else:
                d = json.loads(lines[-1])
                res[name] = {k: d[k] for k in SECONDARY_KEYS if k in d}
        except subprocess.TimeoutExpired:
            res[name] = {"error": f"timeout after {SECONDARY_TIMEOUT_S} s"}
        res[name]["wall_s"] = round(time.time() - t0, 1)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None,
                    choices=sorted(CONFIGS) + ["c3tc", "c4", "c5", "difficulty", "sim",
                                               "baselines"],
                    help="default: c2 (BASELINE.json configs[1]; weak-scaled, one GPU's "
                         "workload per rank, when N > 1); c3 / c3t1 / c3mlp strong-scale "
                         "their 1024 requests over the N GPUs (configs[2])")
    ap.add_argument("--shards", type=int, default=None,
                    help="independent request shards (engines on separate CUDA streams) per "
                         "GPU; default 2 for c2 / c3 / c3t1, 1 otherwise")
    ap.add_argument("--e2e-upload", default="auto", choices=["auto", "gather", "dma", "mixed"],
                    help="e2e input path: DMA runs of the survivor rows (C2: 0.201-0.205 "
                         "M branch-steps/s), the SM gather of the host mapping (0.189-0.195), "
                         "one shard each (0.197-0.200); auto = DMA for windows >= 128 KB")
    ap.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                    help="replay the round loop as a CUDA graph (one buffer rotation per "
                         "graph); auto = on for the launch-bound c1")
    ap.add_argument("--k1-every", type=int, default=8,
                    help="bracket K1 with CUDA events on every N-th timed step (1 shard)")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--slots", type=int, default=None,
                    help="tests only: override the config's request slots (pool scaled)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-gate", action="store_true",
                    help="do not enqueue the timed steps behind the launch gate (profilers)")
    ap.add_argument("--secondary", default=None,
                    help="comma-separated configs measured after the headline and embedded "
                         "in its line under 'secondary' (one subprocess each, bounded); "
                         f"default on the plain N = 1 run: {','.join(SECONDARY)}; 'none' skips")
    args = ap.parse_args()
    default_run = args.config is None
    if args.config is None:
        args.config = "c2"
    cfg = CONFIGS.get(args.config)
    if args.slots and cfg is not None:
        CONFIGS[args.config] = cfg = dict(cfg, R=args.slots, pool=max(8 * args.slots, 64))
    if args.shards is None:
        # two request shards per GPU on two streams hide each shard's round
        # kernel under the other's scoring
        args.shards = 2 if args.config in ("c2", "c2nokv", "c3", "c3t1") else 1
        # (c3mlp: one shard — the tensor-core kernels are persistent, one CTA per SM)
    args.graph = args.graph == "on" or (args.graph == "auto" and args.config == "c1")
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
    else:
        out = run_serving(args, cfg, rank, world, local_rank)
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
        names = (SECONDARY if args.secondary is None and default_run and world == 1
                 else [] if args.secondary in (None, "none")
                 else [x for x in args.secondary.split(",") if x])
        if names:
            # the other BASELINE configs, measured by this same driver-run command
            # (each in its own process: C3 alone holds ~100 GB of activation slabs,
            # so this process first hands its cached device memory back)
            import gc

            import torch
            gc.collect()
            torch.cuda.empty_cache()
            print(f"secondary configs: {torch.cuda.memory_reserved() / 2**30:.2f} GiB still "
                  f"reserved by the headline process", file=sys.stderr)
            out["secondary"] = run_secondary(names)
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
