python tools/spmm_bench.py 2>&1 | grep variant
ENS_SPMM_TILES=1 timeout 120 python tools/spmm_bench.py 2>&1 | tail -3
ENS_SPMM_TILES=1 ENS_TILE_STAGES=2 timeout 120 python tools/spmm_bench.py 2>&1 | grep variant
ENS_SPMM_TILES=1 ENS_TILE_STAGES=4 timeout 120 python tools/spmm_bench.py 2>&1 | grep variant
ENS_SPMM_TILES=1 ENS_TILE_STAGES=2 ENS_TILE_CAP=48 timeout 120 python tools/spmm_bench.py 2>&1 | grep variant
