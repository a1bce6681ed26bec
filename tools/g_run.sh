python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in C2 C4 C3; do
  timeout 900 python bench.py --case $c --steps 20 --warmup 3 --always-steps 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b_$c.json 2> gpurun_out/b_$c.err
  python -c "
import json; d=json.load(open('gpurun_out/b_$c.json')); print('$c', 'ms/step %.3f'%d['ms_per_step'], 'value %.0f'%d['value'], 'iters', d['krylov_iters_per_step'], 'nfact', d['preconditioner']['factorizations_in_timed_steps'])"
done
