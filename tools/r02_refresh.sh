#!/bin/bash
# End-of-round-2 refresh of the bench lines and the bench launch list (the kernels of the apply / SpMM are
# unchanged since tools/r02_profiles.sh was run; this re-measures what changed: e2e path, clock sampler).
set -u
O=gpurun_out
python bench.py --steps 20 --warmup 5 > $O/r02_bench_c2.json 2> $O/r02_bench_c2.err
python bench.py --case C4 --steps 40 --always-steps 5 --e2e-steps 0 > $O/r02_bench_C4.json 2>/dev/null
python bench.py --case C3 --steps 40 --always-steps 3 --e2e-steps 0 > $O/r02_bench_C3.json 2>/dev/null
python tools/step_kernels.py > $O/r02_step_kernels.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file $O/r02_launches_bench.csv \
    python bench.py --steps 5 --warmup 5 --no-cpu-baseline --e2e-steps 3 --always-steps 0 --full-run 0 > /dev/null 2>&1
python bench.py --impl reference --steps 20 --warmup 5 > $O/r02_bench_reference_arm.json 2>/dev/null
echo done
