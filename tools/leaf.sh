for lf in 24 48 96; do echo leaf $lf; ENS_LEAF=$lf timeout 200 python tools/diag_perf.py 2>&1 | grep -E "factor pivot=0|precond|step"; done
