"""Warm in-situ per-level solve timings (ENS_NO_GRAPH=1 ENS_SOLVE_TIMING=1); not a bench."""
import os
import sys

os.environ["ENS_NO_GRAPH"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2108_05110_b200 as P
from paper_2108_05110_b200 import stepper as ST
from paper_2108_05110_b200.engine import _dptr
from paper_2108_05110_b200 import _native as N

disc, cfg, prob = P.build_case(os.environ.get("CASE", "C2"))
eng = ST.get_engine(disc, cfg)
eng.load_state(prob.initial_v, prob.initial_w, None, None)
eng.step(cfg.dt, prob.forcing, prob.boundary)
torch.cuda.synchronize()
X = eng.X[eng.cur]
Z = torch.zeros_like(X)
for _ in range(3):
    N.check(eng.lib.ens_precond_apply(eng.ctx, eng.sptr, _dptr(X), _dptr(Z)), "p")
torch.cuda.synchronize()
dfo = os.environ.get("ENS_DF_PROBE_OUT")
if dfo and hasattr(eng.lib, "ens_df_probe_dump"):    # DF_PROBE build
    eng.lib.ens_df_probe_dump(b"/dev/null")
    N.check(eng.lib.ens_precond_apply(eng.ctx, eng.sptr, _dptr(X), _dptr(Z)), "p")
    print("df probe records", eng.lib.ens_df_probe_dump(dfo.encode()))
out = os.environ.get("ENS_PROBE_OUT")
if out and hasattr(eng.lib, "ens_probe_dump"):      # SG_PROBE build: one clean solve, then dump
    eng.lib.ens_probe_dump(b"/dev/null")
    N.check(eng.lib.ens_precond_apply(eng.ctx, eng.sptr, _dptr(X), _dptr(Z)), "p")
    print("probe records", eng.lib.ens_probe_dump(out.encode()))
os.environ["ENS_SOLVE_TIMING"] = "1"
N.check(eng.lib.ens_precond_apply(eng.ctx, eng.sptr, _dptr(X), _dptr(Z)), "p")
torch.cuda.synchronize()
