"""Aggregate an ncu `--page source --csv --print-source cuda,sass` export per CUDA source line.

    ncu -i rep --page source --csv --print-source cuda,sass > k.csv
    python tools/ncu_lines.py k.csv [topN]
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]
si = h.index("Warp Stall Sampling (All Samples)")
ie = h.index("Instructions Executed")
agg = defaultdict(lambda: [0, 0, ""])
cur = None
for r in rows[hi + 1:]:
    if len(r) <= ie or r[0] in ("Line No", "File Path", "Function Name"):
        continue
    if r[0]:
        cur = (int(r[0]), r[1].strip()[:100])
        continue
    if cur is None:
        continue
    try:
        s, n = int(r[si] or 0), int(r[ie] or 0)
    except ValueError:
        continue
    a = agg[cur[0]]
    a[0] += s
    a[1] += n
    a[2] = cur[1]
S = sum(v[0] for v in agg.values()) or 1
I = sum(v[1] for v in agg.values()) or 1
print(f"samples {S}  warp-instructions {I}")
for ln, (s, n, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100 * s / S:5.1f}%  inst {100 * n / I:5.1f}%  L{ln:<4d} {src}")
