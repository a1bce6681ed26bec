#!/bin/bash
set -u
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/v_smi.txt 2>&1
( time timeout 1500 python -m pytest tests -m gpu -x -q ) > $O/v_pytest.log 2>&1
echo "pytest rc=$?" >> $O/v_pytest.log
timeout 600 python bench.py > $O/v_bench.json 2> $O/v_bench.err
echo "bench rc=$?" >> $O/v_bench.err
# (compute-sanitizer is closed on this GPU pool: see profiles/r02_checks.md for the bounds-checked build instead)
python -c "import __graft_entry__ as g; g.smoke()" > $O/v_smoke.log 2>&1
echo "smoke rc=$?" >> $O/v_smoke.log
