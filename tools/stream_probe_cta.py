"""Per-CTA consumer timeline of ONE launch of the streamed apply (diagnostic build, tools/build_probe.sh).

    TARGET=26 CASE=C2 python tools/stream_probe_cta.py
Marks (consumer warp 0, lane 0): 0 kernel entry, 1 descriptors + first metadata loaded, 2 dependency wait over,
3 first stage full, 4 last unit's mainloop done, 5 epilogue done.  Printed relative to the launch's first entry.
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["ENS_LIB"] = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                     "paper_2108_05110_b200", os.environ.get("PROBE_LIB", "libensmhd_b200_probe.so"))
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
lib.ens_stream_probe_dump.argtypes = [ctypes.c_char_p]
for tgt in [int(x) for x in os.environ.get("TARGET", "26").split(",")]:
    lib.ens_stream_probe_reset()
    lib.ens_stream_probe_target(tgt)
    eng.precond(R, out=Z)
    torch.cuda.synchronize()
    lib.ens_stream_probe_dump(b"/tmp/stp.txt")
    a = np.loadtxt("/tmp/stp.txt")
    if os.environ.get("RAW"):
        np.savetxt(f"gpurun_out/stp_{tgt}.txt", a[a[:, 1] > 0], fmt="%d")
    a = a[(a[:, 1] > 0) & (a[:, 6] > 0)][:, 1:]
    if not len(a):
        print("launch", tgt, "no marks")
        continue
    t0 = a[:, 0].min()
    r = (a - t0) / 1e3
    names = ["entry", "meta", "dep", "full0", "main", "end"]
    print(f"launch {tgt}: {len(a)} CTAs")
    for k, n in enumerate(names):
        print(f"  {n:6s} min {r[:, k].min():7.2f} median {np.median(r[:, k]):7.2f} max {r[:, k].max():7.2f}")
    d = np.diff(r, axis=1)
    for k in range(5):
        print(f"  {names[k]}->{names[k+1]:6s} median {np.median(d[:, k]):7.2f} max {d[:, k].max():7.2f}")
