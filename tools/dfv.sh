for mb in 4 3; do
ENS_NVCC_EXTRA="-DDF_MINB=$mb" python -m paper_2108_05110_b200.build --force > /dev/null
echo minb $mb; timeout 120 python tools/solve_timing.py 2>&1 | tail -1; timeout 120 python tools/diag_perf.py 2>&1 | grep -E "precond"
done
python -m paper_2108_05110_b200.build --force > /dev/null
timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
