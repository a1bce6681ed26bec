"""Summarise an SG_PROBE dump: per solve launch, CTA start spread and phase medians (us)."""
import sys

import numpy as np

a = np.array([list(map(int, l.split()[1:])) for l in open(sys.argv[1]) if l.startswith("probe ")], dtype=np.int64)
# launches are separated in time: sort by start, split where a new kernel begins (gap in key or start jump)
a = a[np.argsort(a[:, 3])]
key = a[:, 0] // 1000000
end = a[:, 3] + a[:, 4:8].sum(1)
cuts = [0]
for i in range(1, len(a)):
    if key[i] != key[i - 1] or a[i, 3] > end[cuts[-1]:i].max():
        cuts.append(i)
cuts.append(len(a))
t_first = a[0, 3]
for c0, c1 in zip(cuts[:-1], cuts[1:]):
    b = a[c0:c1]
    e = end[c0:c1]
    st = (b[:, 3] - b[:, 3].min()) / 1e3
    tag = b[:, 0] % 1000
    last = b[tag == 2]
    print(f"bwd={b[0,0]//1000000} kcmax={((b[:,0]//1000)%1000).max():3d} ctas={len(b):5d} at={(b[:,3].min()-t_first)/1e3:7.1f} "
          f"span={(e.max()-b[:,3].min())/1e3:6.1f} start p50/max={np.median(st):5.1f}/{st.max():5.1f} "
          f"desc={np.median(b[:,4])/1e3:4.1f} gather={np.median(b[:,5])/1e3:4.1f} mma={np.median(b[:,6])/1e3:4.1f} "
          f"epi={np.median(b[:,7])/1e3:4.1f} last={np.median(last[:,7])/1e3 if len(last) else 0:4.1f} "
          f"cta p50/max={np.median((e-b[:,3]))/1e3:5.1f}/{(e-b[:,3]).max()/1e3:5.1f}")
