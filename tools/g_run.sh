for i in 1 2; do
ENS_SPMM_MERGE=0 python tools/spmm_bench.py 2>&1 | grep variant | sed 's/^/merge0 /'
python tools/spmm_bench.py 2>&1 | grep variant | sed 's/^/merge1 /'
done
ENS_SPMM_MERGE=0 python tools/step_ab.py 2>&1 | tail -1
python tools/step_ab.py 2>&1 | tail -1
