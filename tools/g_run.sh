for i in 1 2; do
ENS_RHS_FUSED=0 python tools/step_ab.py 2>&1 | tail -1
python tools/step_ab.py 2>&1 | tail -1
done
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
