"""One preconditioner apply (both systems) inside cudaProfilerStart/Stop, after warm steps: for
`ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum`."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2108_05110_b200 as P
from paper_2108_05110_b200 import stepper as ST

disc, cfg, prob = P.build_case(os.environ.get("CASE", "C2"))
eng = ST.get_engine(disc, cfg)
eng.load_state(prob.initial_v, prob.initial_w, None, None)
t = 0.0
for _ in range(3):
    t += cfg.dt
    eng.step(t, prob.forcing, prob.boundary)
X = eng.X[eng.cur]
Z = torch.zeros_like(X)
eng.precond(X, out=Z)
torch.cuda.synchronize()
torch.cuda.profiler.start()
eng.precond(X, out=Z)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
p = eng.hm.plan
print("nnz_lu", p.stats["nnz_lu"], "algorithmic factor bytes (both systems)", 2 * 8 * p.stats["nnz_lu"])
