cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for r in 1 2; do
python tools/exp_step.py experiments/lib_exp_main.so --reps=7
python tools/exp_step.py - --reps=7
python tools/exp_step.py experiments/lib_exp_main.so 1 "1<<36" --reps=20
python tools/exp_step.py - 1 "1<<36" --reps=20
python tools/exp_step.py experiments/lib_exp_main.so 1 1400000000 --reps=50
python tools/exp_step.py - 1 1400000000 --reps=50
done
