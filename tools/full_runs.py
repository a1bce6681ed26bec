"""Full-length BASELINE runs through the public run() API (one GPU): C2 (100 steps), C3 (500, s = 1),
C4 (1000, delta = 0.1) and C5's per-GPU shard (J = 128 of 1024, 50 steps).  Prints one JSON object
per case: ms/step of the run loop (RunReport.wall_clock, setup excluded, _record diagnostics every
step included), preconditioner rebuilds, max residual, final energy and, for the manufactured
solution, the relative L2 error of the nodal v against the exact field at t_end.

    python tools/full_runs.py [C2 C3 C4 C5]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2108_05110_b200 as P
from paper_2108_05110_b200 import stepper as ST
from paper_2108_05110_b200.problems import BaselineMms

CASES = {"C2": {}, "C3": dict(coupling=1.0), "C4": dict(delta=0.1), "C5": dict(J=128)}

for name in (sys.argv[1:] or list(CASES)):
    t0 = time.perf_counter()
    disc, cfg, prob = P.build_case(name, **CASES[name])
    report, state, _ = P.run(cfg, prob)
    torch.cuda.synchronize()
    eng = ST.get_engine(disc, cfg)
    wall = report.wall_clock[1:]
    out = {"case": name, "members": cfg.num_members, "steps": int(len(wall)), "n_total_dofs": int(disc.n_total),
           "ms_per_step": float(1e3 * wall.mean()), "member_steps_per_s": float(cfg.num_members / wall.mean()),
           "rebuilds": int(eng.n_factor), "max_residual": float(report.residuals[1:].max()),
           "energy_t_end": float(report.energy[-1]), "finite": bool(np.isfinite(report.energy).all()),
           "total_s": round(time.perf_counter() - t0, 1)}
    if name in ("C2", "C5"):
        ex = BaselineMms().exact_v(cfg.t_end, disc, cfg)
        out["rel_l2_error_v_vs_exact"] = float(np.linalg.norm(state.v - ex) / np.linalg.norm(ex))
    print(json.dumps(out), flush=True)
    del eng, state, report
    disc._cache.clear()
    torch.cuda.empty_cache()
