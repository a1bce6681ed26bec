"""Time the pieces of the public advance() loop with numpy state in/out (not a bench)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2108_05110_b200 as P
from paper_2108_05110_b200 import stepper as ST
from paper_2108_05110_b200.ensemble import EnsembleState

disc, cfg, prob = P.build_case("C2")
J = cfg.num_members
st = EnsembleState(v=np.asarray(prob.initial_v), w=np.asarray(prob.initial_w),
                   q=np.zeros((J, disc.n_pres)), r=np.zeros((J, disc.n_pres)))
eng = ST.get_engine(disc, cfg)
tl, ts, tf = [], [], []
host = st
for it in range(12):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng.load_state(host.v, host.w, host.q, host.r)
    t1 = time.perf_counter()
    new, _ = ST._step(eng, host, cfg, prob.forcing, prob.boundary)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    host = EnsembleState(v=new.v, w=new.w, q=new.q, r=new.r, step=new.step, time=new.time)
    t3 = time.perf_counter()
    tl.append(t1 - t0); ts.append(t2 - t1); tf.append(t3 - t2)
    print(f"step {it}: load {1e3*(t1-t0):6.2f} ms  step {1e3*(t2-t1):6.2f} ms  fetch {1e3*(t3-t2):6.2f} ms  iters {eng.last_iters} prev_valid {eng.prev_valid}")
