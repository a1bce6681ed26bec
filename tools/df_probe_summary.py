"""Summarise a DF_PROBE dump: per sweep span, CTA busy vs waiting, task durations by kind."""
import sys

import numpy as np

a = np.array([list(map(int, l.split())) for l in open(sys.argv[1])], dtype=np.uint64)
key = a[:, 0]
bwd = (key >> np.uint64(62)).astype(int)
cta = ((key >> np.uint64(40)) & np.uint64((1 << 22) - 1)).astype(int)
item = (key & np.uint64((1 << 32) - 1)).astype(int)
t0, t1, t2 = a[:, 1].astype(np.int64), a[:, 2].astype(np.int64), a[:, 3].astype(np.int64)
for d in (0, 1):
    s = bwd == d
    if not s.any():
        continue
    T0, T1, T2, C, I = t0[s], t1[s], t2[s], cta[s], item[s]
    span = (T2.max() - T0.min()) / 1e3
    wait = (T1 - T0) / 1e3
    work = (T2 - T1) / 1e3
    nct = len(np.unique(C))
    print(f"{'bwd' if d else 'fwd'}: tasks {s.sum()}  ctas {nct}  span {span:.1f} us  "
          f"sum wait {wait.sum():.0f} us  sum work {work.sum():.0f} us  (busy frac {work.sum() / (nct * span):.2f})")
    print(f"   wait p50/p90/max {np.median(wait):.2f}/{np.percentile(wait, 90):.2f}/{wait.max():.1f}  "
          f"work p50/p90/max {np.median(work):.2f}/{np.percentile(work, 90):.2f}/{work.max():.1f}")
    # timeline in 10 buckets: how many tasks running
    o = np.argsort(I)
    for lo, hi in [(0, 0.1), (0.1, 0.25), (0.25, 0.5), (0.5, 0.75), (0.75, 1.0)]:
        n = len(I)
        sel = o[int(lo * n):int(hi * n)]
        print(f"   items {lo:.2f}-{hi:.2f}: start {(T0[sel].min() - T0.min()) / 1e3:7.1f}..{(T2[sel].max() - T0.min()) / 1e3:7.1f} us "
              f"wait p50 {np.median(wait[sel]):.2f}  work p50 {np.median(work[sel]):.2f}")
