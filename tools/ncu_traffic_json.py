"""ncu --csv metrics dump (dram__bytes_read.sum, dram__bytes_write.sum, gpu__time_duration.sum) ->
the per-kernel traffic JSON bench.py reads for roofline.traffic (profiles/r02_*_traffic.json).

    python tools/ncu_traffic_json.py in.csv out.json "<kernel description>" "<command>" <algorithmic bytes> "<note>"
"""
import csv
import json
import sys
from collections import OrderedDict

src, dst, kernel, command, alg, note = sys.argv[1:7]
rows = list(csv.reader(open(src)))
hdr, data = None, OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        data.setdefault((int(d["ID"]), name), {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
per = OrderedDict()
for (_, name), m in data.items():
    e = per.setdefault(name, dict(launches=0, dram_read_bytes=0.0, dram_write_bytes=0.0, time_ns=0.0))
    e["launches"] += 1
    e["dram_read_bytes"] += m.get("dram__bytes_read.sum", 0.0)
    e["dram_write_bytes"] += m.get("dram__bytes_write.sum", 0.0)
    e["time_ns"] += m.get("gpu__time_duration.sum", 0.0)
tot = int(sum(e["dram_read_bytes"] + e["dram_write_bytes"] for e in per.values()))
json.dump(dict(kernel=kernel, command=command, per_kernel=per, traffic_bytes_per_launch=tot,
               algorithmic_bytes=int(float(alg)), note=note), open(dst, "w"), indent=1)
print(dst, tot, "bytes,", round(tot / float(alg), 3), "x algorithmic")
