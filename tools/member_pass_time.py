"""Warm time of the fused right-hand-side element pass (ens_rhs_fused: k_member_pass<true> + k_member_gather<true>),
CUDA events on the engine stream (diagnostic builds: ENS_LIB=...)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

import paper_2108_05110_b200 as P
from paper_2108_05110_b200.engine import Engine

disc, cfg, prob = P.build_case(os.environ.get("CASE", "C2"))
eng = Engine(disc, cfg)
eng.load_state(prob.initial_v, prob.initial_w, None, None)
eng.compute_means()
X = eng.X[eng.cur]
with eng.on_stream():
    for _ in range(3):
        eng._rhs_and_member_pass(X, None)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(10):
            eng._rhs_and_member_pass(X, None)
        torch.cuda.synchronize()
for e in prof.key_averages():
    if "member" in e.key:
        print(f"{os.environ.get('ENS_LIB', 'default')[-24:]:24s} {e.key[:40]:40s} {e.device_time_total / e.count:8.1f} us")
