#!/bin/bash
# diagnostic build of the library with the streamed-solve timeline probe (tools/stream_probe.py)
cd "$(dirname "$0")/../paper_2108_05110_b200" && nvcc -DST_PROBE -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC -shared -I../include -o libensmhd_b200_probe.so csrc/*.cu -lcudart 2>&1 | grep -i "error" ; exit 0
