for w in 1 0; do
ENS_SOLVE_CW64=$w timeout 1500 python bench.py --case C5 --steps 4 --warmup 3 --always-steps 0 --e2e-steps 0 > gpurun_out/bench_C5_$w.json 2> gpurun_out/bench_C5_$w.err
python -c "
import json; d=json.load(open('gpurun_out/bench_C5_$w.json')); print('cw64=$w', round(d['value']), round(d['ms_per_step'],2), 'apply %.2f ms %.1f TF frac %.3f'%(d['roofline']['ms_per_launch'], d['roofline']['achieved'], d['roofline']['frac']))"
done
