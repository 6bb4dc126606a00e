"""Aggregate ncu warp-stall samples per CUDA source line:
    python tools/ncu_lines.py report.ncu-rep [top_n]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur_file, hdr, agg, total = None, None, {}, 0.0
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr) or not r[0]:
        continue
    try:
        v = float(r[4] or 0)
    except ValueError:
        continue
    total += v
    key = (cur_file, int(r[0]))
    agg[key] = (agg.get(key, (0, ""))[0] + v, r[1].strip()[:100])
print(f"total stall samples {total:.0f}")
for (f, ln), (v, src) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{v:7.0f} {100 * v / max(total, 1):5.1f}%  {f}:{ln:<5d} {src}")
