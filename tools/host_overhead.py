"""Host (Python) time per step vs device time per step; not a bench."""
import os
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
for _ in range(6):
    t += cfg.dt
    eng.step(t, prob.forcing, prob.boundary)
torch.cuda.synchronize()
import cProfile, pstats
pr = cProfile.Profile()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(eng.stream)
h0 = time.perf_counter()
pr.enable()
for _ in range(20):
    t += cfg.dt
    eng.step(t, prob.forcing, prob.boundary)
pr.disable()
h1 = time.perf_counter()
b.record(eng.stream)
torch.cuda.synchronize()
print(f"host {1e3 * (h1 - h0) / 20:.3f} ms/step (includes waits)  device {a.elapsed_time(b) / 20:.3f} ms/step")
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
