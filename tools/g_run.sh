set -e; python -m paper_2108_05110_b200.build > /dev/null; set +e
for kf in fgmres richardson; do
  for c in C2 C4 C3; do
    ENS_KRYLOV_FIRST=$kf timeout 900 python bench.py --case $c --steps 10 --warmup 3 --always-steps 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b_${kf}_$c.json 2> gpurun_out/b_${kf}_$c.err
    python -c "
import json; d=json.load(open('gpurun_out/b_${kf}_$c.json')); print('$kf $c', 'ms/step %.3f'%d['ms_per_step'], 'value %.0f'%d['value'], 'iters', d['krylov_iters_per_step'], 'nfact', d['preconditioner']['factorizations_in_timed_steps'])"
  done
done
