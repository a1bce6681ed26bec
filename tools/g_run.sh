python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo c2=$?
ncu --set full --import-source on --clock-control none -k regex:k_spmm_ -s 4 -c 2 -o gpurun_out/spmm_c2 python tools/spmm_bench.py > gpurun_out/ncu_spmm.log 2>&1; echo ncu=$?
timeout 1500 python bench.py --case C5 --steps 3 --warmup 3 --always-steps 0 --e2e-steps 0 > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err; echo C5=$?
tail -2 gpurun_out/bench_C5.err; head -c 1500 gpurun_out/bench_C5.json
