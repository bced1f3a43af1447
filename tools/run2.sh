cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_parity.py -x -q -k "oracle_random or large_goldens or escalation or golden" 2>&1 | tail -2
for r in 1 2; do
python tools/exp_step.py experiments/lib_exp_base.so --reps=5
python tools/exp_step.py experiments/lib_exp_ck.so --reps=5
done
