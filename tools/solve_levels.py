"""One preconditioner application bracketed by cudaProfilerStart/Stop, for
`ncu --profile-from-start off` per-level launch lists (not a bench)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2108_05110_b200 as P
from paper_2108_05110_b200 import stepper as ST
from paper_2108_05110_b200.engine import _dptr
from paper_2108_05110_b200 import _native as N

case = os.environ.get("CASE", "C2")
disc, cfg, prob = P.build_case(case)
eng = ST.get_engine(disc, cfg)
eng.load_state(prob.initial_v, prob.initial_w, None, None)
eng.step(cfg.dt, prob.forcing, prob.boundary)
torch.cuda.synchronize()
X = eng.X[eng.cur]
Z = torch.zeros_like(X)
N.check(eng.lib.ens_precond_apply(eng.ctx, eng.sptr, _dptr(X), _dptr(Z)), "p")
torch.cuda.synchronize()
torch.cuda.profiler.start()
N.check(eng.lib.ens_precond_apply(eng.ctx, eng.sptr, _dptr(X), _dptr(Z)), "p")
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
