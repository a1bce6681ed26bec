"""GPU timeline of the public advance() call with numpy state in/out (torch.profiler); not a bench.

Prints, for each of the last advance() calls, every device activity (copies and kernels) with its
start relative to the call and its duration, and the idle time between them."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

import paper_2108_05110_b200 as P
from paper_2108_05110_b200.ensemble import EnsembleState

disc, cfg, prob = P.build_case(os.environ.get("CASE", "C2"))
J = cfg.num_members
host = EnsembleState(v=np.asarray(prob.initial_v), w=np.asarray(prob.initial_w),
                     q=np.zeros((J, disc.n_pres)), r=np.zeros((J, disc.n_pres)))
for _ in range(8):
    new, _ = P.advance(host, cfg, disc, prob.forcing, prob.boundary)
    host = EnsembleState(v=new.v, w=new.w, q=new.q, r=new.r, step=new.step, time=new.time)
torch.cuda.synchronize()
n = 3
marks = []
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(n):
        t0 = time.perf_counter()
        new, _ = P.advance(host, cfg, disc, prob.forcing, prob.boundary)
        t1 = time.perf_counter()
        host = EnsembleState(v=new.v, w=new.w, q=new.q, r=new.r, step=new.step, time=new.time)
        t2 = time.perf_counter()
        marks.append((t1 - t0, t2 - t1))
    torch.cuda.synchronize()
path = os.environ.get("TRACE", "gpurun_out/e2e_trace.json")
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
k = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")], key=lambda e: e["ts"])
for a, f in marks:
    print(f"advance {1e3 * a:.3f} ms   fetch {1e3 * f:.3f} ms")
# last call: everything after the last but one big D2H group
big = [i for i, e in enumerate(k) if e.get("cat") == "gpu_memcpy" and "DtoH" in e["name"] and e["dur"] > 100]
start = big[-5] + 1 if len(big) >= 5 else 0
t0 = k[start]["ts"]
prev_end = t0
small = 0.0
for e in k[start:]:
    gap = e["ts"] - prev_end
    if e["dur"] > 8 or gap > 8:
        print(f"{e['ts'] - t0:9.1f} us  dur {e['dur']:8.1f}  gap {gap:7.1f}  {e['name'].split('(')[0][:60]}")
    else:
        small += e["dur"]
    prev_end = max(prev_end, e["ts"] + e["dur"])
print(f"last call span {prev_end - t0:.1f} us; activities under 8 us not listed: {small:.1f} us")
