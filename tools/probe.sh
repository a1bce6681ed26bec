# diagnostic: rebuild with SG_PROBE, dump per-CTA solve phase timestamps, rebuild the normal library
ENS_NVCC_EXTRA=-DSG_PROBE python -m paper_2108_05110_b200.build --force > /dev/null
ENS_PROBE_OUT=gpurun_out/probe.log python tools/solve_timing.py > gpurun_out/probe_run.log 2>&1
python -m paper_2108_05110_b200.build --force > /dev/null
