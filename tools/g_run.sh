timeout 1500 python bench.py --case C5 --steps 5 --warmup 3 --always-steps 0 --e2e-steps 0 > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err; echo C5=$?
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo c2=$?
