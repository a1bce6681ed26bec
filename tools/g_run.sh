for i in 1 2; do
ENS_LIB=$PWD/paper_2108_05110_b200/libensmhd_b200_old.so python tools/step_ab.py 2>&1 | tail -1
python tools/step_ab.py 2>&1 | tail -1
done
