"""Host-side cost of warm graphed time steps (cProfile, sorted by own time); not a bench."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2108_05110_b200 as P
from paper_2108_05110_b200 import stepper as ST

disc, cfg, prob = P.build_case(os.environ.get("CASE", "C2"))
eng = ST.get_engine(disc, cfg)
eng.load_state(prob.initial_v, prob.initial_w, None, None)
t = 0.0
for _ in range(5):
    t += cfg.dt
    eng.step(t, prob.forcing, prob.boundary)
torch.cuda.synchronize()
n = 40
t0 = time.perf_counter()
pr = cProfile.Profile()
pr.enable()
for _ in range(n):
    t += cfg.dt
    eng.step(t, prob.forcing, prob.boundary)
pr.disable()
print(f"wall per step {(time.perf_counter() - t0) / n * 1e3:.3f} ms (under cProfile)")
pstats.Stats(pr).sort_stats("tottime").print_stats(18)

if os.environ.get("E2E") == "1":     # the public advance() loop with host arrays in / out
    import numpy as np
    from paper_2108_05110_b200.ensemble import EnsembleState
    J = cfg.num_members
    host = EnsembleState(v=np.asarray(prob.initial_v), w=np.asarray(prob.initial_w),
                         q=np.zeros((J, disc.n_pres)), r=np.zeros((J, disc.n_pres)))
    for _ in range(8):
        new, _ = P.advance(host, cfg, disc, prob.forcing, prob.boundary)
        host = EnsembleState(v=new.v, w=new.w, q=new.q, r=new.r, step=new.step, time=new.time)
    pr = cProfile.Profile()
    t0 = time.perf_counter()
    pr.enable()
    for _ in range(n):
        new, _ = P.advance(host, cfg, disc, prob.forcing, prob.boundary)
        host = EnsembleState(v=new.v, w=new.w, q=new.q, r=new.r, step=new.step, time=new.time)
    pr.disable()
    print(f"advance loop: wall per step {(time.perf_counter() - t0) / n * 1e3:.3f} ms (under cProfile)")
    pstats.Stats(pr).sort_stats("tottime").print_stats(35)
