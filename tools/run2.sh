cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for r in 1 2; do
python tools/exp_step.py experiments/lib_exp_main.so --reps=5
python tools/exp_step.py - --reps=5
done
python tools/exp_step.py - 1 1400000000 --reps=100
python tools/exp_step.py - 1 "1<<36" --reps=30
python tools/exp_step.py - "(1<<50)-(1<<40)+1" "1<<50" --reps=10
