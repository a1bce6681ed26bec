"""One saddle SpMM (both systems) inside cudaProfilerStart/Stop after warm steps, for ncu traffic
captures (`--profile-from-start off --cache-control none --metrics dram__bytes_read.sum,...`)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2108_05110_b200 as P
from paper_2108_05110_b200 import stepper as ST
from paper_2108_05110_b200 import _native as N
from paper_2108_05110_b200.engine import _dptr, spmm_bytes

disc, cfg, prob = P.build_case(os.environ.get("CASE", "C2"))
eng = ST.get_engine(disc, cfg)
eng.load_state(prob.initial_v, prob.initial_w, None, None)
t = 0.0
for _ in range(3):
    t += cfg.dt
    eng.step(t, prob.forcing, prob.boundary)
X = eng.X[eng.cur]
Y = torch.empty_like(X)
for _ in range(3):
    N.check(eng.lib.ens_spmm(eng.ctx, eng.sptr, _dptr(eng.as_vals), _dptr(X), None, _dptr(Y), 0), "spmm")
torch.cuda.synchronize()
torch.cuda.profiler.start()
N.check(eng.lib.ens_spmm(eng.ctx, eng.sptr, _dptr(eng.as_vals), _dptr(X), None, _dptr(Y), 0), "spmm")
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("algorithmic SpMM bytes (both systems)", spmm_bytes(eng.hm, eng.J))
