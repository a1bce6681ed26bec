for c in C2 C4 C3; do
for r in 0 1; do
  ENS_ROUND_FACTOR=$r timeout 900 python bench.py --case $c --steps 20 --warmup 3 --always-steps 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b_$c.json 2> gpurun_out/b_$c.err
  python -c "
import json; d=json.load(open('gpurun_out/b_$c.json')); print('round $r $c', 'ms/step %.3f'%d['ms_per_step'], 'iters', d['krylov_iters_per_step'], 'nfact', d['preconditioner']['factorizations_in_timed_steps'])"
done; done
