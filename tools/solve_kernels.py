"""Warm, graph-mode kernel sequence of one preconditioner application (CUPTI via torch.profiler)."""
import os
import sys

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
X = eng.X[eng.cur]
Z = torch.zeros_like(X)
for _ in range(3):
    N.check(eng.lib.ens_precond_apply(eng.ctx, eng.sptr, _dptr(X), _dptr(Z)), "p")
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    N.check(eng.lib.ens_precond_apply(eng.ctx, eng.sptr, _dptr(X), _dptr(Z)), "p")
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
tot = 0.0
for e in ev:
    d = e.time_range.end - e.time_range.start
    tot += d
    print(f"{e.time_range.start - t0:8.1f} {d:7.1f} us  {e.name[:60]}")
print(f"sum {tot:.1f} us  span {ev[-1].time_range.end - t0:.1f} us")
