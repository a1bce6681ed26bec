"""A/B of the factorisation: warm time (CUDA events) and a bitwise fingerprint of one preconditioner
apply with the new factors (ENS_LIB selects the library build)."""
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
for _ in range(2):
    t += cfg.dt
    eng.step(t, prob.forcing, prob.boundary)
eng.factor()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(eng.stream):
    a.record()
    for _ in range(5):
        eng.factor()
    b.record()
torch.cuda.synchronize()
torch.manual_seed(0)
R = torch.randn_like(eng.X[eng.cur])
Z = torch.zeros_like(R)
eng.precond(R, out=Z)
torch.cuda.synchronize()
print(f"{os.path.basename(os.environ.get('ENS_LIB', 'current'))} {case}: factor {a.elapsed_time(b) / 5:.2f} ms "
      f"fingerprint {int(Z.view(torch.int64).sum().item())}")
