"""Warm factorisation kernels attributed to (tree level, op) via the launch schedule (CUPTI).

CASE=C4 python tools/factor_levels.py   -> per-level / per-op device time of one factorisation.
The kernels of one ens_factor run in schedule order (OP_ZERO is a memset, empty OP_ORIG
ranges launch nothing), so event i maps to the i-th launching schedule row.
"""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

import paper_2108_05110_b200 as P
from paper_2108_05110_b200 import stepper as ST
from paper_2108_05110_b200.engine import _dptr
from paper_2108_05110_b200 import _native as N

OPS = {0: "zero", 1: "orig", 2: "extadd", 3: "diag", 4: "hpanel", 5: "update", 6: "gpanel"}

case = os.environ.get("CASE", "C2")
disc, cfg, prob = P.build_case(case)
eng = ST.get_engine(disc, cfg)
eng.load_state(prob.initial_v, prob.initial_w, None, None)
eng.step(cfg.dt, prob.forcing, prob.boundary)
for _ in range(2):
    N.check(eng.lib.ens_factor(eng.ctx, eng.sptr, _dptr(eng.as_vals), None), "f")
torch.cuda.synchronize()
reps = int(os.environ.get("REPS", "3"))
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(reps):
        N.check(eng.lib.ens_factor(eng.ctx, eng.sptr, _dptr(eng.as_vals), None), "f")
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and "memset" not in e.name.lower()
      and "Memset" not in e.name]
ev.sort(key=lambda e: e.time_range.start)
plan = eng.hm.plan
sched = plan.schedule["factor"]
orig_off = plan.orig_level_off
rows = []
for r in sched:
    op, L = int(r[0]), int(r[1])
    if op == 0:
        continue
    if op == 1 and orig_off[L + 1] <= orig_off[L]:
        continue
    rows.append((op, L, int(r[3])))
per = len(ev) // reps
print(f"{case}: {len(ev)} kernels, {per} per factorisation, schedule rows {len(rows)} (+stream pack)")
agg = defaultdict(float)
lvl = defaultdict(float)
opt = defaultdict(float)
span = []
for rep in range(reps):
    seg = ev[rep * per:(rep + 1) * per]
    span.append(seg[-1].time_range.end - seg[0].time_range.start)
    for i, e in enumerate(seg):
        d = e.time_range.end - e.time_range.start
        if i < len(rows):
            op, L, n = rows[i]
            agg[(L, OPS[op])] += d / reps
            lvl[L] += d / reps
            opt[OPS[op]] += d / reps
        else:
            agg[("pack", e.name.split("(")[0][:24])] += d / reps
            opt["pack"] += d / reps
print(f"span per factorisation {np.mean(span):.1f} us, kernel sum {sum(opt.values()):.1f} us")
for k, v in sorted(opt.items(), key=lambda kv: -kv[1]):
    print(f"  {k:8s} {v:9.1f} us")
fm, fk = plan.f_m.astype(np.int64), plan.f_k.astype(np.int64)
for L in range(plan.nlevels):
    lo, hi = plan.level_front_off[L], plan.level_front_off[L + 1]
    gf = 2 * (2 * fm[lo:hi] ** 2 * fk[lo:hi]).sum() / 1e9
    parts = "  ".join(f"{o}={agg.get((L, o), 0):7.1f}" for o in ("extadd", "diag", "hpanel", "update", "gpanel"))
    print(f"L{L:2d} nf {hi-lo:5d} mmax {fm[lo:hi].max():5d} {lvl[L]:8.1f} us  {gf:6.2f} GF  "
          f"{gf / max(lvl[L], 1e-9) * 1e3:6.2f} TF/s | {parts}")
