"""Warm time of one factorisation of both shared matrices (CUDA events on the engine stream).

    CASE=C3 python tools/factor_time.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2108_05110_b200 as P
from paper_2108_05110_b200 import stepper as ST

case = os.environ.get("CASE", "C2")
disc, cfg, prob = P.build_case(case)
eng = ST.get_engine(disc, cfg)
eng.load_state(prob.initial_v, prob.initial_w, None, None)
eng.step(cfg.dt, prob.forcing, prob.boundary)
for _ in range(2):
    eng.factor()
torch.cuda.synchronize()
ts = []
for _ in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(eng.stream):
        a.record()
        eng.factor()
        b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ts.sort()
print(f"{case}: factorisation {ts[len(ts) // 2]:.3f} ms (min {ts[0]:.3f}), lib {os.environ.get('ENS_LIB', 'default')}")
