for fl in "-DSG_PROBE -DSG_NOB" "-DSG_PROBE -DSG_NOA" "-DSG_PROBE -DSG_NOA -DSG_NOB"; do
ENS_NVCC_EXTRA="$fl" python -m paper_2108_05110_b200.build --force > /dev/null
ENS_SOLVE_STAGES=2 ENS_PROBE_OUT=gpurun_out/probe_$(echo $fl | tr -d ' -').log python tools/solve_timing.py > /dev/null 2>&1
done
python -m paper_2108_05110_b200.build --force > /dev/null
