"""Host-side cost of the pieces between two advance() calls with numpy state in / out (not a bench)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2108_05110_b200 as P
from paper_2108_05110_b200 import stepper as ST
from paper_2108_05110_b200.ensemble import EnsembleState

disc, cfg, prob = P.build_case(os.environ.get("CASE", "C2"))
J = cfg.num_members
host = EnsembleState(v=np.asarray(prob.initial_v), w=np.asarray(prob.initial_w),
                     q=np.zeros((J, disc.n_pres)), r=np.zeros((J, disc.n_pres)))
for _ in range(8):
    new, _ = P.advance(host, cfg, disc, prob.forcing, prob.boundary)
    host = EnsembleState(v=new.v, w=new.w, q=new.q, r=new.r, step=new.step, time=new.time)
acc = {}


def lap(name, t0):
    t1 = time.perf_counter()
    acc[name] = acc.get(name, 0.0) + (t1 - t0)
    return t1


n = 30
for _ in range(n):
    torch.cuda.synchronize()
    t = time.perf_counter()
    eng = ST.get_engine(disc, cfg)
    t = lap("get_engine", t)
    ds = ST._device_state_of(host, eng)
    t = lap("_device_state_of", t)
    eng.load_state(host.v, host.w, host.q, host.r)
    t = lap("load_state (enqueue)", t)
    new, _ = ST._step(eng, host, cfg, prob.forcing, prob.boundary, fetch=True)
    t = lap("_step (incl. waiting for the solve)", t)
    v = new.v
    t = lap("new.v (incl. waiting for the download)", t)
    w, q, r = new.w, new.q, new.r
    t = lap("new.w, q, r", t)
    host = EnsembleState(v=v, w=w, q=q, r=r, step=new.step, time=new.time)
    t = lap("EnsembleState(...)", t)
for k, v in acc.items():
    print(f"{k:45s} {1e6 * v / n:9.1f} us")
