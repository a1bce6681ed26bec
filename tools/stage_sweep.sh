for st in 2 3 4 5; do echo "stages $st"; ENS_SOLVE_STAGES=$st timeout 200 python tools/solve_kernels.py 2>&1 | grep -v Warn | grep -E "k_sgemm|sum" | awk '{print $2}' | tr '\n' ' '; echo; done
