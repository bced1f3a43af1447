cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_parity.py -x -q -k "pattern13 or large_goldens or batch_and_pipeline" 2>&1 | tail -3
for r in 1 2; do
python tools/exp_step.py experiments/lib_exp_main.so --reps=5
python tools/exp_step.py - --reps=5
done
for it in 7 8 9 10 11; do
  printf "item %s: " $it; SQF2K_MED_ITEM=$it SQF2K_MED_BIAS=0.25 python tools/exp_step.py - --reps=5 | sed 's/^ *[a-z_.0-9]*: //'
done
python tools/exp_time.py - "(1<<50)-(1<<44)+1" "1<<50"
