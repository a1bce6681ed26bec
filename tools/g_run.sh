python -m pytest tests -m gpu -x -q -k "graphs or c1_matches or refactor or case_runs" 2>&1 | tail -3
python tools/step_gaps.py 2>&1 | grep -v Warn | head -12
ENS_STEP_GRAPH=0 python tools/step_gaps.py 2>&1 | grep -v Warn | head -3
python bench.py --no-cpu-baseline --always-steps 0 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo c2=$?
head -c 400 gpurun_out/bench_c2.json; grep -o '"gpu_launches": [0-9]*' gpurun_out/bench_c2.json
tail -3 gpurun_out/bench_c2.err
