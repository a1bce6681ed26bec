"""Summarise an ncu SASS source export: top instructions by stall samples + stall totals.

    ncu -i rep --page source --csv -k regex:K -c 1 --print-source sass > k.csv
    python tools/ncu_hot.py k.csv [topN]
"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = rows[2:]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
si = h.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
tot = Counter()
lines = []
for r in data:
    try:
        s = int(r[si])
    except (ValueError, IndexError):
        continue
    lines.append((s, r[0][-5:], r[1].strip()))
    for i in stall_cols:
        try:
            tot[h[i]] += int(r[i])
        except ValueError:
            pass
S = sum(s for s, _, _ in lines) or 1
print("total samples", S)
print("stalls:", ", ".join(f"{k[6:]}={100 * v / S:.1f}%" for k, v in tot.most_common(8)))
for s, a, src in sorted(lines, reverse=True)[:top]:
    print(f"{100 * s / S:5.1f}%  {a}  {src}")
