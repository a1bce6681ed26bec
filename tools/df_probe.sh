# diagnostic: dataflow-solve task timeline (DF_PROBE build), then rebuild the normal library
ENS_NVCC_EXTRA=-DDF_PROBE python -m paper_2108_05110_b200.build --force > /dev/null
ENS_DF_PROBE_OUT=gpurun_out/dfprobe.log python tools/solve_timing.py > gpurun_out/dfprobe_run.log 2>&1
python -m paper_2108_05110_b200.build --force > /dev/null
