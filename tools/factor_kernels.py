"""Warm, graph-mode kernel sequence of one factorisation (CUPTI via torch.profiler), grouped by op."""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

import paper_2108_05110_b200 as P
from paper_2108_05110_b200 import stepper as ST
from paper_2108_05110_b200.engine import _dptr
from paper_2108_05110_b200 import _native as N

disc, cfg, prob = P.build_case(os.environ.get("CASE", "C2"))
eng = ST.get_engine(disc, cfg)
eng.load_state(prob.initial_v, prob.initial_w, None, None)
eng.step(cfg.dt, prob.forcing, prob.boundary)
for _ in range(2):
    N.check(eng.lib.ens_factor(eng.ctx, eng.sptr, _dptr(eng.as_vals), None), "f")
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    N.check(eng.lib.ens_factor(eng.ctx, eng.sptr, _dptr(eng.as_vals), None), "f")
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
agg = defaultdict(lambda: [0, 0.0])
tot = 0.0
for e in ev:
    d = e.time_range.end - e.time_range.start
    k = e.name.split("(")[0][:40]
    agg[k][0] += 1
    agg[k][1] += d
    tot += d
span = ev[-1].time_range.end - ev[0].time_range.start
print(f"kernels {len(ev)}  sum {tot:.1f} us  span {span:.1f} us")
for k, (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{us:9.1f} us  {c:5d}  {k}")
t0 = ev[0].time_range.start
for e in ev[:40] + ev[-24:]:
    print(f"{e.time_range.start - t0:9.1f} {e.time_range.end - e.time_range.start:8.1f}  {e.name.split('(')[0][:30]}")
# time per launch sequence position (top levels = later launches)
n = len(ev)
for q in range(10):
    seg = ev[q * n // 10:(q + 1) * n // 10]
    print(f"decile {q}: {sum(e.time_range.end - e.time_range.start for e in seg):8.1f} us in {len(seg)} launches")
