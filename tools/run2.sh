cd $GRAFT_REPO_ROOT
for r in 1 2; do
for v in cur d11 d11dyn8 dyn8 d11dyn8m2 d11dyn8s5 d11dyn16; do python tools/exp_step.py experiments/lib_exp_$v.so 1 1400000000 --reps=100 2>&1 | tail -1; done
done
for v in cur d11 d11dyn8; do python tools/exp_step.py experiments/lib_exp_$v.so --reps=4 2>&1 | tail -1; python tools/exp_step.py experiments/lib_exp_$v.so 1 "1<<36" --reps=20 2>&1 | tail -1; done
