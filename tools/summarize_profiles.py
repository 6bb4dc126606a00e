"""Summarise a profile pass (tools/profile_all.sh) into profiles/<tag>/ text files."""
import csv
import collections
import json
import os
import subprocess
import sys

tag = sys.argv[1]
src = f"gpurun_out/prof_{tag}"
dst = f"profiles/{tag}"
os.makedirs(dst, exist_ok=True)
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__occupancy_limit_registers",
        "lts__t_sector_hit_rate.pct", "sm__cycles_active.avg", "gpc__cycles_elapsed.max"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units, vals = rows[0], rows[1], rows[2]
    return {n: (vals[i], units[i]) for i, n in enumerate(h)}


summary = {}
for name in ("k1_full", "k1rows_full", "round_full", "kv_full", "k3_full", "k4_full", "tc_full",
             "mlp1_full", "mlp2_full", "step_full"):
    rep = f"{src}/{name}.ncu-rep"
    if not os.path.exists(rep):
        continue
    r = raw(rep)
    pick = {k: r[k] for k in KEYS if k in r}
    summary[name] = {"kernel": r.get("Kernel Name", ("?", ""))[0], **{k: f"{v} {u}" for k, (v, u) in pick.items()}}
    det = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True).stdout
    with open(f"{dst}/{name}_details.txt", "w") as f:
        f.write(det)
    lines = subprocess.run([sys.executable, "tools/ncu_lines.py", rep, "25"], capture_output=True,
                           text=True).stdout
    with open(f"{dst}/{name}_hot_lines.txt", "w") as f:
        f.write(lines)
with open(f"{dst}/ncu_full_summary.json", "w") as f:
    json.dump(summary, f, indent=1)

UNIT = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6,
        "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6,
        "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3,
        "B": 1e-6, "KB": 1e-3, "MB": 1.0, "GB": 1e3}


STEP_KERNELS = ("score_", "round_kernel", "kv_round_kernel", "mlp_probe_tc", "linear_kernel")


def launch_list(csv_name: str, title: str) -> None:
    """Per-kernel summary of an ncu launch list (us, MB; units from the CSV)."""
    path = f"{src}/{csv_name}.csv"
    if not os.path.exists(path):
        return
    rows = list(csv.reader(open(path)))
    hdr, data = None, collections.defaultdict(dict)
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            v = float(d["Metric Value"].replace(",", "")) * UNIT.get(d["Metric Unit"], 1.0)
            data[(int(d["ID"]), d["Kernel Name"])][d["Metric Name"]] = v
    agg = collections.defaultdict(list)
    for (_i, k), m in sorted(data.items()):
        agg[k.split("(")[0]].append(m)
    tot = sum(m["gpu__time_duration.sum"] for ms in agg.values() for m in ms)
    # share of the serving step: the per-round kernels only (setup fills, the e2e
    # pass's host gathers and the read-only peak probe excluded)
    is_step = {k: any(s in k for s in STEP_KERNELS) for k in agg}
    step_tot = sum(m["gpu__time_duration.sum"] for k, ms in agg.items() if is_step[k] for m in ms)
    with open(f"{dst}/{csv_name}_summary.txt", "w") as f:
        f.write(title + "\n")
        f.write(f"{'kernel':55s} {'n':>4s} {'mean_us':>9s} {'min_us':>8s} {'max_us':>8s} "
                f"{'rd_MB':>9s} {'wr_MB':>8s} {'share':>6s} {'step':>6s}\n")
        for k, ms in sorted(agg.items(), key=lambda x: -sum(m["gpu__time_duration.sum"] for m in x[1])):
            t = [m["gpu__time_duration.sum"] for m in ms]
            rd = [m.get("dram__bytes_read.sum", 0) for m in ms]
            wr = [m.get("dram__bytes_write.sum", 0) for m in ms]
            f.write(f"{k[:55]:55s} {len(t):4d} {sum(t)/len(t):9.2f} {min(t):8.2f} {max(t):8.2f} "
                    f"{sum(rd)/len(rd):9.2f} {sum(wr)/len(wr):8.2f} {sum(t)/tot:6.1%} "
                    + (f"{sum(t)/step_tot:6.1%}" if is_step[k] else f"{'-':>6s}") + "\n")
    os.system(f"cp {path} {dst}/{csv_name}.csv")
    print(open(f"{dst}/{csv_name}_summary.txt").read())


launch_list("launches_c2", "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
            "dram__bytes_write.sum --clock-control none  python bench.py --steps 8 --warmup 3 "
            "(cold-cache, serialised: compare shares, not absolutes)")
launch_list("launches_c3mlp", "the same for python bench.py --config c3mlp --steps 4 --warmup 2")
launch_list("launches_difficulty", "ncu --metrics gpu__time_duration.sum, the classifier's "
            "kernels in python bench.py --config difficulty (normalise, 3 layers, head)")
print(json.dumps(summary, indent=1))
