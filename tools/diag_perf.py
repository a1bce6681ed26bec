"""Quick per-phase timings on the GPU (CUDA events on the engine stream); not a bench."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2108_05110_b200 as P
from paper_2108_05110_b200 import stepper as ST
from paper_2108_05110_b200.engine import _dptr
from paper_2108_05110_b200 import _native as N

case = os.environ.get("CASE", "C2")
disc, cfg, prob = P.build_case(case)
eng = ST.get_engine(disc, cfg)
eng.load_state(prob.initial_v, prob.initial_w, None, None)
t = 0.0
for _ in range(3):
    t += cfg.dt
    eng.step(t, prob.forcing, prob.boundary)
torch.cuda.synchronize()
print("after steps: pivoting", eng.pivoting, "last_pert", eng.last_pert, "iters", eng.last_iters, "nfactor", eng.n_factor)
s = eng.stream


def tcall(fn, reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    a.record(s)
    for _ in range(reps):
        fn()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


X = eng.X[eng.cur]
Y = torch.empty_like(X)
Z = torch.zeros_like(X)
sp = tcall(lambda: N.check(eng.lib.ens_spmm(eng.ctx, eng.sptr, _dptr(eng.as_vals), _dptr(X), None, _dptr(Y), 0), "s"), 50)
print(f"spmm {sp*1e3:.1f} us  (ENS_SPMM_ITER={os.environ.get('ENS_SPMM_ITER', '1')})")
for piv in (0, 1):
    eng.lib.ens_set_pivoting(eng.ctx, piv)
    npert = N.I32(0)
    f = tcall(lambda: N.check(eng.lib.ens_factor(eng.ctx, eng.sptr, _dptr(eng.as_vals), None), "f"), 5)
    N.check(eng.lib.ens_factor(eng.ctx, eng.sptr, _dptr(eng.as_vals), N.C.byref(npert)), "f")
    print(f"factor pivot={piv}: {f:.2f} ms  npert={npert.value}")
sv = tcall(lambda: N.check(eng.lib.ens_precond_apply(eng.ctx, eng.sptr, _dptr(X), _dptr(Z)), "p"), 10)
print(f"precond apply {sv*1e3:.1f} us")
st = tcall(lambda: eng._step(t + cfg.dt, prob.forcing, prob.boundary), 5)
print(f"step {st:.2f} ms  iters {eng.last_iters}")
