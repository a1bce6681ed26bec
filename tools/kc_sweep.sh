for cfg in "-DSG_MINB=3" "-DSG_MINB=4" "-DSG_KC=16 -DSG_MINB=4" "-DSG_KC=16 -DSG_MINB=3"; do
ENS_NVCC_EXTRA="$cfg" python -m paper_2108_05110_b200.build --force > /dev/null
for st in 2 3; do echo "cfg $cfg stages $st"; ENS_SOLVE_STAGES=$st timeout 200 python tools/solve_kernels.py 2>&1 | grep -v Warn | grep -E "sum"; done
done
python -m paper_2108_05110_b200.build --force > /dev/null
