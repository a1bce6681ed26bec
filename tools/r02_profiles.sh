#!/bin/bash
# Round-2 measurement set (run on the B200 box from the repo root; outputs under gpurun_out/).
set -u
O=gpurun_out
python bench.py > $O/r02_bench_c2.json 2> $O/r02_bench_c2.err
python bench.py --impl reference > $O/r02_bench_reference_arm.json 2>/dev/null
python bench.py --case C4 --steps 40 --always-steps 5 --e2e-steps 0 > $O/r02_bench_C4.json 2>/dev/null
python bench.py --case C3 --steps 40 --always-steps 3 --e2e-steps 0 > $O/r02_bench_C3.json 2>/dev/null
# launch list of the bench command itself (cold, serialised per-kernel times: shares, not absolutes)
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/r02_launches_bench.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 --always-steps 0 --full-run 0 > /dev/null 2>&1
# warm DRAM traffic of one preconditioner apply and one SpMM (no cache flush between kernels)
ncu --profile-from-start off --cache-control none --clock-control none \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
    python tools/precond_once.py > $O/r02_apply_traffic.csv 2>/dev/null
ncu --profile-from-start off --cache-control none --clock-control none \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
    python tools/spmm_once.py > $O/r02_spmm_traffic.csv 2>/dev/null
# full capture of the largest streamed-GEMM launch (leaf level, backward) for the stall / source pages
ncu --profile-from-start off --set full --import-source on -k regex:k_stream_gemm --launch-skip 20 -c 1 \
    -o $O/r02_stream_gemm python tools/precond_once.py > /dev/null 2>&1
ncu --profile-from-start off --set full --import-source on -k regex:k_spmm -c 1 \
    -o $O/r02_spmm python tools/spmm_once.py > /dev/null 2>&1
echo done
