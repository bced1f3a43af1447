cd $GRAFT_REPO_ROOT
for r in 1 2; do for v in "$@"; do python tools/exp_step.py experiments/lib_exp_$v.so --reps=7; done; done
