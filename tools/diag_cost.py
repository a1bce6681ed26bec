"""Cost of the per-step _record diagnostics (energy, member norms, divergence) at C2 (not a bench)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2108_05110_b200 as P
from paper_2108_05110_b200 import stepper as ST

disc, cfg, prob = P.build_case(os.environ.get("CASE", "C2"))
eng = ST.get_engine(disc, cfg)
eng.load_state(prob.initial_v, prob.initial_w, None, None)
t = 0.0
for _ in range(6):
    t += cfg.dt
    eng.step(t, prob.forcing, prob.boundary)
torch.cuda.synchronize()
n = 20
t0 = time.perf_counter()
for _ in range(n):
    eng.diagnostics()
torch.cuda.synchronize()
d = (time.perf_counter() - t0) / n
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(eng.stream):
    a.record()
    for _ in range(n):
        eng.means_valid = False
        eng._compute_means()
        N = eng.lib
        from paper_2108_05110_b200 import _native as NN
        from paper_2108_05110_b200.engine import _dptr
        NN.check(N.ens_diagnostics(eng.ctx, eng.sptr, _dptr(eng.X[eng.cur]), _dptr(eng.means), _dptr(eng.diag_out)), "d")
    b.record()
torch.cuda.synchronize()
print(f"diagnostics(): {d * 1e3:.3f} ms wall per call; device {a.elapsed_time(b) / n * 1e3:.1f} us per call")
