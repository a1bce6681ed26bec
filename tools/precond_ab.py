"""A/B of the preconditioner apply: bitwise fingerprint + warm time (ENS_LIB selects the library build)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2108_05110_b200 as P
from paper_2108_05110_b200 import stepper as ST

case = os.environ.get("CASE", "C2")
disc, cfg, prob = P.build_case(case)
eng = ST.get_engine(disc, cfg)
eng.load_state(prob.initial_v, prob.initial_w, None, None)
t = 0.0
for _ in range(3):
    t += cfg.dt
    eng.step(t, prob.forcing, prob.boundary)
torch.manual_seed(0)
R = torch.randn_like(eng.X[eng.cur])
Z = torch.zeros_like(R)
eng.precond(R, out=Z)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(eng.stream):
    a.record()
    for _ in range(20):
        eng.precond(R, out=Z)
    b.record()
torch.cuda.synchronize()
print(f"{os.path.basename(os.environ.get('ENS_LIB', 'current'))} {case}: apply {a.elapsed_time(b) / 20 * 1e3:.1f} us "
      f"fingerprint {int(Z.view(torch.int64).sum().item())}")
