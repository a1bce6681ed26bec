"""Summarise an ncu --csv metrics dump: per-kernel time and DRAM bytes, grouped by kernel name."""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        data.setdefault((int(d["ID"]), d["Kernel Name"].split("(")[0]), {})[d["Metric Name"]] = \
            float(d["Metric Value"].replace(",", ""))
tot = 0.0
per = OrderedDict()
for (i, name), m in data.items():
    t = m.get("gpu__time_duration.sum", 0.0) / 1e3
    tot += t
    b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    per.setdefault(name, [0, 0.0, 0.0])
    per[name][0] += 1
    per[name][1] += t
    per[name][2] += b
    if "-v" in sys.argv:
        print(f"{i:4d} {name[:40]:40s} {t:8.1f} us {b / 1e6:8.1f} MB")
for name, (n, t, b) in per.items():
    print(f"{name[:50]:50s} n={n:3d} {t:9.1f} us {b / 1e6:9.1f} MB  {b / max(t, 1e-9) / 1e3:7.1f} GB/s")
print(f"total {tot:.1f} us")
