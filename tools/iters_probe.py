import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2108_05110_b200 as P
from paper_2108_05110_b200 import stepper as ST
disc, cfg, prob = P.build_case("C2")
for policy in ("always", "adaptive"):
    for guess in ("extrapolate", "previous"):
        ST.set_solver_options(refactor=policy, guess=guess)
        eng = ST.get_engine(disc, cfg)
        eng.load_state(prob.initial_v, prob.initial_w, None, None)
        t = 0.0; its = []
        for _ in range(8):
            t += cfg.dt
            eng.step(t, prob.forcing, prob.boundary)
            its.append(eng.last_iters)
        print(policy, guess, its, flush=True)
