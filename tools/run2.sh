cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_parity.py -x -q -k "pattern13 or large_goldens or full_range" 2>&1 | tail -2
for r in 1 2; do
python tools/exp_step.py experiments/lib_exp_cur.so --reps=4 2>&1 | tail -1
python tools/exp_step.py - --reps=4 2>&1 | tail -1
done
