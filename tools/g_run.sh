for i in 1 2; do
ENS_LIB=$PWD/paper_2108_05110_b200/libensmhd_b200_old.so python tools/step_ab.py 2>&1 | tail -1
ENS_LIB=$PWD/paper_2108_05110_b200/libensmhd_b200_b.so python tools/step_ab.py 2>&1 | tail -1
python tools/step_ab.py 2>&1 | tail -1
done
ncu --metrics gpu__time_duration.sum -k regex:k_member_pass -c 3 python tools/step_ab.py 2>&1 | grep -E "k_member_pass|duration" | head -6
ENS_LIB=$PWD/paper_2108_05110_b200/libensmhd_b200_b.so ncu --metrics gpu__time_duration.sum -k regex:k_member_pass -c 3 python tools/step_ab.py 2>&1 | grep -E "duration" | head -3
