"""SpMM micro-timing on the engine stream (CUDA events), warm and after an L2 flush; prints a bitwise fingerprint.

    ENS_SPMM_P=<variant> CASE=C2 python tools/spmm_bench.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2108_05110_b200 as P
from paper_2108_05110_b200 import stepper as ST
from paper_2108_05110_b200 import _native as N
from paper_2108_05110_b200.engine import _dptr

case = os.environ.get("CASE", "C2")
over = {}
if "J" in os.environ:
    over["J"] = int(os.environ["J"])
disc, cfg, prob = P.build_case(case, **over)
eng = ST.get_engine(disc, cfg)
eng.load_state(prob.initial_v, prob.initial_w, None, None)
t = 0.0
for _ in range(2):
    t += cfg.dt
    eng.step(t, prob.forcing, prob.boundary)
torch.cuda.synchronize()
s = eng.stream
X = eng.X[eng.cur]
torch.manual_seed(0)
B = torch.randn_like(X)
Y = torch.empty_like(X)
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=X.device)


def run(mode):
    N.check(eng.lib.ens_spmm(eng.ctx, eng.sptr, _dptr(eng.as_vals), _dptr(X), _dptr(B) if mode else None, _dptr(Y),
                             mode), "spmm")


def timed(mode, reps, cold):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    run(mode)
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        for a, b in ev:
            if cold:
                flush.fill_(1.0)
            a.record()
            run(mode)
            b.record()
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) * 1e3 for a, b in ev)
    return ts[len(ts) // 2]


for mode in (0, 1):
    w = timed(mode, 50, False)
    c = timed(mode, 20, True)
    run(mode)
    torch.cuda.synchronize()
    fp = int(Y.view(torch.int64).sum().item())
    print(f"variant {os.environ.get('ENS_SPMM_P', '0')} tiles {os.environ.get('ENS_SPMM_TILES', '0')}:{os.environ.get('ENS_TILE_STAGES', '3')}:{os.environ.get('ENS_TILE_CAP', '-')} J={cfg.num_members} mode {mode}: warm {w:.1f} us  "
          f"cold {c:.1f} us  fingerprint {fp}")
