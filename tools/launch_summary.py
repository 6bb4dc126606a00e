"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list:
per kernel name, launches and mean / max duration (us).
    python tools/launch_summary.py launches.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, agg = None, collections.defaultdict(list)
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(d["Metric Unit"], 1.0)
            agg[d["Kernel Name"].split("(")[0][:70]].append(float(d["Metric Value"]) * scale)
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{k:70s} n={len(v):5d} mean={sum(v) / len(v):9.2f} us max={max(v):9.2f} "
          f"share={sum(v) / tot:6.1%}")
