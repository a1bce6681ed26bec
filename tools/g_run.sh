ENS_LIB=$PWD/paper_2108_05110_b200/libensmhd_b200_old.so python tools/precond_ab.py 2>&1 | tail -1
python tools/precond_ab.py 2>&1 | tail -1
CASE=C4 python tools/precond_ab.py 2>&1 | tail -1
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py --no-cpu-baseline --always-steps 0 --e2e-steps 0 2>/dev/null | head -c 250
