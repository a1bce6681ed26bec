python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/gpu_tests.log
python bench.py --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo c2=$?
for c in C4 C3; do
  timeout 900 python bench.py --case $c --steps 5 --warmup 3 --always-steps 2 --e2e-steps 0 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo $c=$?
done
timeout 1500 python bench.py --case C5 --steps 3 --warmup 3 --always-steps 0 --e2e-steps 0 > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err; echo C5=$?
tail -3 gpurun_out/bench_C5.err
