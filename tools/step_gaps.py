"""Idle gaps between the kernels of warm time steps (torch.profiler chrome trace); not a bench.

Prints per-step busy/idle time and the largest gaps with the kernels on either side."""
import json
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

import paper_2108_05110_b200 as P
from paper_2108_05110_b200 import stepper as ST

case = os.environ.get("CASE", "C2")
n = int(os.environ.get("STEPS", "5"))
disc, cfg, prob = P.build_case(case)
comm = None
if os.environ.get("FORCE_DIST") == "1":   # sharded code path on one rank (run under torchrun)
    import torch.distributed as dist
    dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
    comm = dist.group.WORLD
eng = ST.get_engine(disc, cfg, comm=comm)
eng.load_state(prob.initial_v, prob.initial_w, None, None)
t = 0.0
for _ in range(6):
    t += cfg.dt
    eng.step(t, prob.forcing, prob.boundary, then=(t + cfg.dt, prob.forcing, prob.boundary))
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(n):
        t += cfg.dt
        eng.step(t, prob.forcing, prob.boundary, then=(t + cfg.dt, prob.forcing, prob.boundary))
    torch.cuda.synchronize()
path = os.environ.get("TRACE", "gpurun_out/step_trace.json")
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
k = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")], key=lambda e: e["ts"])
busy = sum(e["dur"] for e in k)
span = k[-1]["ts"] + k[-1]["dur"] - k[0]["ts"]
print(f"{case}: {n} steps, span {span / n:.1f} us/step, kernels busy {busy / n:.1f} us/step, "
      f"idle {(span - busy) / n:.1f} us/step, {len(k) / n:.1f} kernels/step")
gaps = defaultdict(lambda: [0, 0.0])
for a, b in zip(k[:-1], k[1:]):
    g = b["ts"] - (a["ts"] + a["dur"])
    if g > 1.5:
        key = f'{a["name"].split("(")[0][:40]} -> {b["name"].split("(")[0][:40]}'
        gaps[key][0] += 1
        gaps[key][1] += g
for key, (c, g) in sorted(gaps.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"{g / n:8.1f} us/step  {c / n:5.1f}/step  {key}")
