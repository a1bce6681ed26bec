for sk in 64 128 192 256; do echo "split $sk"; ENS_SPLIT_K=$sk timeout 200 python tools/solve_kernels.py 2>&1 | grep -v Warn | grep -E "k_sgemm|sum" | awk '{print $2}' | tr '\n' ' '; echo; done
