"""BASELINE parameter variants through run(): C3 with s = 0.01 and 0.1 (500 steps), C4 with delta = 0.01
(1000 steps).  One JSON object per run (same fields as tools/full_runs.py)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2108_05110_b200 as P
from paper_2108_05110_b200 import stepper as ST

for name, over in (("C3", dict(coupling=0.01)), ("C3", dict(coupling=0.1)), ("C4", dict(delta=0.01))):
    t0 = time.perf_counter()
    disc, cfg, prob = P.build_case(name, **over)
    report, state, _ = P.run(cfg, prob)
    torch.cuda.synchronize()
    eng = ST.get_engine(disc, cfg)
    wall = report.wall_clock[1:]
    print(json.dumps({"case": name, **over, "members": cfg.num_members, "steps": int(len(wall)),
                      "ms_per_step": float(1e3 * wall.mean()), "member_steps_per_s": float(cfg.num_members / wall.mean()),
                      "rebuilds": int(eng.n_factor), "max_residual": float(report.residuals[1:].max()),
                      "energy_t_end": float(report.energy[-1]), "finite": bool(np.isfinite(report.energy).all()),
                      "total_s": round(time.perf_counter() - t0, 1)}), flush=True)
    del eng, state, report
    disc._cache.clear()
    torch.cuda.empty_cache()
