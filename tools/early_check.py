"""Does the announced-step path enqueue the next pre-solve graph behind the solve (diagnostic)?"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2108_05110_b200 as P
from paper_2108_05110_b200 import stepper as ST

disc, cfg, prob = P.build_case(os.environ.get("CASE", "C2"))
eng = ST.get_engine(disc, cfg)
eng.load_state(prob.initial_v, prob.initial_w, None, None)
calls = []
orig = eng._replay


def spy(g):
    calls.append(g)
    return orig(g)


eng._replay = spy
t = 0.0
for i in range(14):
    t += cfg.dt
    n0 = len(calls)
    eng.step(t, prob.forcing, prob.boundary, then=(t + cfg.dt, prob.forcing, prob.boundary))
    print(i, "replays", len(calls) - n0, "ones", eng._ones, "wb1", eng._wb[1] is not None, "spec", eng._spec is not None,
          "iters", eng.last_iters)
torch.cuda.synchronize()
for mode in ("then", "plain"):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(eng.stream)
    for i in range(20):
        t += cfg.dt
        if mode == "then":
            eng.step(t, prob.forcing, prob.boundary, then=(t + cfg.dt, prob.forcing, prob.boundary))
        else:
            eng.step(t, prob.forcing, prob.boundary)
    b.record(eng.stream)
    torch.cuda.synchronize()
    print(mode, a.elapsed_time(b) / 20, "ms/step")
