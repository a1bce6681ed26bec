"""Summarise an ncu `--metrics gpu__time_duration.sum --csv` launch list: per-kernel launches, time, share.

    python tools/launch_summary.py launches.csv [--skip N]   (skip the first N launches, e.g. setup)
"""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
skip = int(sys.argv[sys.argv.index("--skip") + 1]) if "--skip" in sys.argv else 0
rows = [r for r in csv.reader(open(path)) if r and r[0].isdigit()]
hdr = next(r for r in csv.reader(open(path)) if r and r[0] == "ID")
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = defaultdict(lambda: [0, 0.0])
for r in rows[skip:]:
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
    name = r[ki].split("(")[0].replace("void ", "")[:48]
    agg[name][0] += 1
    agg[name][1] += float(r[vi].replace(",", "")) * scale
tot = sum(v[1] for v in agg.values())
print(f"{len(rows) - skip} launches, {tot:.1f} us total")
print("| kernel | launches | total us | share |\n|---|---|---|---|")
for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"| `{k}` | {n} | {us:.1f} | {100 * us / tot:.1f} % |")
