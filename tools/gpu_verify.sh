#!/bin/bash
set -u
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/v_smi.txt 2>&1
( time timeout 1500 python -m pytest tests -m gpu -x -q ) > $O/v_pytest.log 2>&1
echo "pytest rc=$?" >> $O/v_pytest.log
timeout 600 python bench.py > $O/v_bench.json 2> $O/v_bench.err
echo "bench rc=$?" >> $O/v_bench.err
timeout 300 compute-sanitizer --tool memcheck python -c "import __graft_entry__ as g; g.smoke()" > $O/v_san.log 2>&1
echo "san rc=$?" >> $O/v_san.log
