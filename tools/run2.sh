cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for r in 1 2; do
python tools/exp_step.py experiments/lib_exp_cur.so --reps=4 2>&1 | tail -1
python tools/exp_step.py - --reps=4 2>&1 | tail -1
done
for w in '1 1400000000' '1 1<<36' '(1<<50)-(1<<40)+1 1<<50'; do
set -- $w
python tools/exp_step.py experiments/lib_exp_cur.so "$1" "$2" --reps=30 2>&1 | tail -1
python tools/exp_step.py - "$1" "$2" --reps=30 2>&1 | tail -1
done
