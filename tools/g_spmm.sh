python -m pytest tests -m gpu -x -q -k "wide or tiles" 2>&1 | tail -2
for J in 64 128; do for w in 0 1 2; do ENS_SPMM_WIDE=$w J=$J python tools/spmm_bench.py 2>&1 | grep variant | sed "s/^/wide=$w /"; done; done
timeout 1500 python bench.py --case C5 --steps 3 --warmup 3 --always-steps 0 --e2e-steps 0 > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err; echo C5=$?
tail -2 gpurun_out/bench_C5.err; head -c 600 gpurun_out/bench_C5.json
