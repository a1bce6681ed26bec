"""A/B of whole time steps: warm ms/step (CUDA events) + bitwise fingerprint of the state (ENS_LIB selects the build)."""
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
for _ in range(4):
    t += cfg.dt
    eng.step(t, prob.forcing, prob.boundary)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
a.record(eng.stream)
n = 16
for _ in range(n):
    t += cfg.dt
    eng.step(t, prob.forcing, prob.boundary)
b.record(eng.stream)
torch.cuda.synchronize()
X = eng.X[eng.cur]
print(f"{os.path.basename(os.environ.get('ENS_LIB', 'current'))} {case}: {a.elapsed_time(b) / n:.3f} ms/step "
      f"fingerprint {int(X.view(torch.int64).sum().item())} factorizations {eng.n_factor}")
