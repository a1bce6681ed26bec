cat > /tmp/steps_only.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2108_05110_b200 as P
from paper_2108_05110_b200 import stepper as ST
disc, cfg, prob = P.build_case("C2")
eng = ST.get_engine(disc, cfg)
eng.load_state(prob.initial_v, prob.initial_w, None, None)
t = 0.0
for _ in range(6):
    t += cfg.dt
    eng.step(t, prob.forcing, prob.boundary)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(5):
    t += cfg.dt
    eng.step(t, prob.forcing, prob.boundary)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("iters", eng.last_iters, "factorizations", eng.n_factor)
PY
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches_step.csv python /tmp/steps_only.py > gpurun_out/ncu_steps.log 2>&1; echo ncu=$?
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench=$?
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
