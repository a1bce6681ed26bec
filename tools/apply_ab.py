"""A/B of the preconditioner apply: classic k_sgemm path (ENS_SOLVE_STREAM=0) vs the streamed path (=1),
same factorisation input, warm CUDA-event timings and the relative difference of the outputs.

    CASE=C2 python tools/apply_ab.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2108_05110_b200 as P
from paper_2108_05110_b200.engine import Engine, apply_bytes, apply_flops

case = os.environ.get("CASE", "C2")
over = json.loads(os.environ.get("OVER", "{}"))
disc, cfg, prob = P.build_case(case, **over)
out = {}
res = {}
rng = np.random.default_rng(5)
for mode in ("0", "1"):
    os.environ["ENS_SOLVE_STREAM"] = mode
    eng = Engine(disc, cfg)
    eng.load_state(prob.initial_v, prob.initial_w, None, None)
    t = 0.0
    for _ in range(2):
        t += cfg.dt
        eng.step(t, prob.forcing, prob.boundary)
    eng.factor()
    R = torch.from_numpy(rng.standard_normal((2, eng.ntot, eng.J))).cuda() if mode == "0" else R
    Z = torch.zeros_like(R)
    for _ in range(3):
        eng.precond(R, out=Z)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(eng.stream)
    for _ in range(20):
        eng.precond(R, out=Z)
    b.record(eng.stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 20
    fa, fb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fa.record(eng.stream)
    for _ in range(3):
        eng.factor()
    fb.record(eng.stream)
    torch.cuda.synchronize()
    out[mode] = Z.cpu().numpy()
    by = apply_bytes(eng.hm, eng.J)
    res[mode] = dict(apply_ms=ms, gbs=by / ms / 1e6, frac=by / ms / 1e6 / 6548.2,
                     tflops=apply_flops(eng.hm, eng.J) / ms / 1e9, factor_ms=fa.elapsed_time(fb) / 3)
    del eng
d = np.linalg.norm(out["1"] - out["0"]) / np.linalg.norm(out["0"])
print(json.dumps(dict(case=case, over=over, classic=res["0"], stream=res["1"], rel_diff=float(d))))
