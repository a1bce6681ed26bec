for i in 1 2; do
ENS_LIB=$PWD/paper_2108_05110_b200/libensmhd_b200_old.so python tools/precond_ab.py 2>&1 | tail -1
python tools/precond_ab.py 2>&1 | tail -1
done
CASE=C4 ENS_LIB=$PWD/paper_2108_05110_b200/libensmhd_b200_old.so python tools/precond_ab.py 2>&1 | tail -1
CASE=C4 python tools/precond_ab.py 2>&1 | tail -1
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
