#!/bin/bash
# one GPU iteration: parity tests, C2/C3/C4 timings, ncu full capture of the tile kernel on C2
# usage (on the box): bash tools/gpu_iter.sh TAG
TAG=${1:-x}
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 400 -p no:cacheprovider -x > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/gpu_tests.log
python tools/prof_verify.py "(1<<50)-(1<<40)+1" "1<<50" --reps 3 | tail -1
python tools/prof_verify.py 1 "1<<36" --reps 3 | tail -1
python tools/prof_verify.py 1 1400000000 --reps 2 > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"tile_kernel" -s 1 -c 1 -o gpurun_out/prof_$TAG python tools/prof_verify.py 1 1400000000 --reps 2 > gpurun_out/ncu.log 2>&1; echo ncu_rc=$?
