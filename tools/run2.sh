cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_parity.py -x -q -k "oracle_random or large_goldens" 2>&1 | tail -2
for r in 1 2; do
python tools/exp_step.py experiments/lib_exp_noalign.so --reps=5
python tools/exp_step.py - --reps=5
done
for it in 7 8 9 10; do
  printf "align item %s: " $it; SQF2K_MED_ITEM=$it SQF2K_MED_BIAS=0.25 python tools/exp_step.py - --reps=5 | sed 's/^ *[a-z_.0-9]*: //'
done
python tools/exp_step.py experiments/lib_exp_noalign.so 1 1400000000 --reps=50
python tools/exp_step.py - 1 1400000000 --reps=50
