ENS_NVCC_EXTRA="-DSG_KMAX=128 -DSG_MINB=4" python -m paper_2108_05110_b200.build --force > /dev/null
echo "kmax128 minb4 split128"; ENS_SPLIT_K=128 timeout 200 python tools/solve_kernels.py 2>&1 | grep -v Warn | grep -E "k_sgemm|sum" | awk '{print $2}' | tr '\n' ' '; echo
ENS_NVCC_EXTRA="-DSG_KMAX=128 -DSG_MINB=3" python -m paper_2108_05110_b200.build --force > /dev/null
echo "kmax128 minb3 split128"; ENS_SPLIT_K=128 timeout 200 python tools/solve_kernels.py 2>&1 | grep -v Warn | grep -E "sum"
python -m paper_2108_05110_b200.build --force > /dev/null
echo "default"; timeout 200 python tools/solve_kernels.py 2>&1 | grep -v Warn | grep -E "k_sgemm|sum" | awk '{print $2}' | tr '\n' ' '; echo
