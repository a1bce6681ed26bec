for mb in 3 4; do
ENS_NVCC_EXTRA="-DSG_MINB=$mb" python -m paper_2108_05110_b200.build --force > /dev/null
echo minb $mb; timeout 200 python tools/solve_kernels.py 2>&1 | grep -v Warn | grep -E "k_sgemm|sum" | awk '{print $2}' | tr '\n' ' '; echo
timeout 200 python tools/diag_perf.py 2>&1 | grep -E "precond"
done
python -m paper_2108_05110_b200.build --force > /dev/null
