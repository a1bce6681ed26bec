"""Timeline probe of the streamed solve (diagnostic build, -DST_PROBE; prebuilt as
libensmhd_b200_probe.so): per launch of one preconditioner apply, first-CTA start and last-CTA end
(globaltimer), so launch spans and the gaps between dependent launches are visible; plus per-CTA
consumer statistics of the first forward GEMM launch.

    ENS_NVCC_EXTRA=-DST_PROBE (build into libensmhd_b200_probe.so), then CASE=C2 python tools/stream_probe.py
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["ENS_LIB"] = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                     "paper_2108_05110_b200", "libensmhd_b200_probe.so")
os.environ["ENS_NO_GRAPH"] = os.environ.get("ENS_NO_GRAPH", "0")
import numpy as np
import torch

import paper_2108_05110_b200 as P
from paper_2108_05110_b200.engine import Engine

disc, cfg, prob = P.build_case(os.environ.get("CASE", "C2"))
eng = Engine(disc, cfg)
eng.load_state(prob.initial_v, prob.initial_w, None, None)
eng.factor()
R = torch.randn(2, eng.ntot, eng.J, dtype=torch.float64, device="cuda")
Z = torch.zeros_like(R)
for _ in range(3):
    eng.precond(R, out=Z)
torch.cuda.synchronize()
lib = eng.lib
lib.ens_stream_probe_levels.argtypes = [ctypes.c_char_p]
lib.ens_stream_probe_dump.argtypes = [ctypes.c_char_p]
lib.ens_stream_probe_reset()
lib.ens_stream_probe_target(int(os.environ.get("TARGET", "2")))
eng.precond(R, out=Z)
torch.cuda.synchronize()
lib.ens_stream_probe_levels(b"/tmp/stl.txt")
lib.ens_stream_probe_dump(b"/tmp/stp.txt")
L = np.loadtxt("/tmp/stl.txt", dtype=np.float64)
L = L[L[:, 2] > 0]
t0 = L[:, 1].min()
prev_end = None
tot_gap = 0.0
for i, a, b in L:
    gap = (a - prev_end) / 1e3 if prev_end is not None else 0.0
    tot_gap += max(gap, 0.0)
    print(f"launch {int(i):3d} start {(a - t0) / 1e3:8.2f} span {(b - a) / 1e3:7.2f} us  gap {gap:6.2f}")
    prev_end = b
a = np.loadtxt("/tmp/stp.txt")
a = a[a[:, 6] > 0]
if len(a):
    body = a[:, 3] / 1e3
    print("per-CTA body us: min %.1f median %.1f max %.1f; wait median %.1f; stages median %d max %d; units max %d"
          % (body.min(), np.median(body), body.max(), np.median(a[:, 4]) / 1e3, np.median(a[:, 5]), a[:, 5].max(),
             a[:, 6].max()))
    prev_end = b
print(f"apply span {(L[:, 2].max() - t0) / 1e3:.1f} us, sum of gaps {tot_gap:.1f} us")
a = np.loadtxt("/tmp/stp.txt")
a = a[a[:, 6] > 0]
if len(a):
    print(f"launch {os.environ.get('TARGET', '2')}: CTAs", len(a), "body median us", np.median(a[:, 3]) / 1e3, "wait median us",
          np.median(a[:, 4]) / 1e3, "stages median", np.median(a[:, 5]), "units median", np.median(a[:, 6]))
