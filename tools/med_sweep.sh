#!/bin/bash
# Medium-schedule sweep on the GPU box: C4 call time per (item, bias) knob
# pair (build_med reads SQF2K_MED_* from the environment).
cd "$(dirname "$0")/.."
W="(1<<50)-(1<<40)+1"
for it in ${ITEMS:-3 3.5 4 4.5 5 5.5 6 6.5 7 8}; do
  for b in ${BIASES:-0 0.25 0.5 0.75}; do
    printf "item %-4s bias %-5s " $it $b
    SQF2K_MED_ITEM=$it SQF2K_MED_BIAS=$b python tools/exp_step.py - "$W" "1<<50" --reps=10 | sed 's/^ *main: //'
  done
done
