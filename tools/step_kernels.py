"""Warm per-kernel breakdown of the time step (torch.profiler / CUPTI); not a bench."""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

import paper_2108_05110_b200 as P
from paper_2108_05110_b200 import stepper as ST

case = os.environ.get("CASE", "C2")
n = int(os.environ.get("STEPS", "5"))
disc, cfg, prob = P.build_case(case)
eng = ST.get_engine(disc, cfg)
eng.load_state(prob.initial_v, prob.initial_w, None, None)
t = 0.0
for _ in range(6):
    t += cfg.dt
    eng.step(t, prob.forcing, prob.boundary, then=(t + cfg.dt, prob.forcing, prob.boundary))
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(n):
        t += cfg.dt
        eng.step(t, prob.forcing, prob.boundary, then=(t + cfg.dt, prob.forcing, prob.boundary))
    torch.cuda.synchronize()
agg = defaultdict(lambda: [0, 0.0])
tot = 0.0
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        k = e.name.split("(")[0][:60]
        agg[k][0] += 1
        agg[k][1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
        tot += agg[k][1] * 0 + (e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total)
print(f"{case}: {n} steps, iters {eng.last_iters}, kernel time/step {tot / n:.1f} us")
for k, (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:30]:
    print(f"{us / n:9.1f} us/step  {c / n:6.1f}/step  {k}")
