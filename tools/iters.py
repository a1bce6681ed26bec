"""FGMRES iteration history per step for a case (CASE env, default C2); not a bench."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2108_05110_b200 as P
from paper_2108_05110_b200 import stepper as ST

case = os.environ.get("CASE", "C2")
nsteps = int(os.environ.get("STEPS", "12"))
for guess in ("previous", "extrapolate"):
    ST.set_solver_options(guess=guess)
    disc, cfg, prob = P.build_case(case)
    eng = ST.get_engine(disc, cfg)
    eng.load_state(prob.initial_v, prob.initial_w, None, None)
    t, hist = 0.0, []
    for _ in range(nsteps):
        t += cfg.dt
        eng.step(t, prob.forcing, prob.boundary)
        hist.append((eng.last_iters, f"{max(eng.last_relres):.1e}", eng.n_factor))
    torch.cuda.synchronize()
    print(case, guess, hist)
