"""Profiling driver: one C2 engine, a few steps, then isolated factor / solve calls.

    python tools/prof_step.py [--case C2] [--what solve|factor|step]
Used under ncu (launch lists / --set full); never a source of bench numbers.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2108_05110_b200 as P
from paper_2108_05110_b200 import stepper as ST

ap = argparse.ArgumentParser()
ap.add_argument("--case", default="C2")
ap.add_argument("--what", default="solve")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--J", type=int, default=None)
a = ap.parse_args()
over = {} if a.J is None else {"J": a.J}
disc, cfg, prob = P.build_case(a.case, **over)
eng = ST.get_engine(disc, cfg)
eng.load_state(prob.initial_v, prob.initial_w, None, None)
t = 0.0
for _ in range(2):
    t += cfg.dt
    eng.step(t, prob.forcing, prob.boundary)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("measure")
X = eng.X[eng.cur]
Z = torch.zeros_like(X)
for _ in range(a.reps):
    if a.what == "solve":
        eng.precond(X, out=Z)
    elif a.what == "factor":
        eng.factor()
    else:
        t += cfg.dt
        eng.step(t, prob.forcing, prob.boundary)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("ok", a.what, eng.hm.plan.stats)
