ENS_SOLVE_DEEP_CTAS=0 python tools/precond_ab.py 2>&1 | tail -1
for st in 3 4 5; do for th in 296 444 888; do
echo -n "stages $st ctas<=$th: "; ENS_SOLVE_DEEP_STAGES=$st ENS_SOLVE_DEEP_CTAS=$th python tools/precond_ab.py 2>&1 | tail -1
done; done
