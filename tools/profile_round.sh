#!/bin/bash
# The round's evidence run (on the GPU box, from the repo root):
#   bash tools/profile_round.sh TAG
# bench lines (C5 headline + C2 secondary + CPU baseline, the reference arm,
# C3 and C4), the paper's [1, 2^50) with clocks, the ncu launch list of the
# bench command, and one `ncu --set full` capture each of tile_fused (one C5
# batch: the 2^38-integer window ending at 2^50) and window_scan (2^37 window).
# Outputs land in gpurun_out/; tools/summarize_round.py turns them into
# profiles/ files.
TAG=${1:-r2}
O=gpurun_out
python bench.py > $O/${TAG}_bench_c5.json 2> $O/${TAG}_bench_c5.err; echo bench_c5=$?
python bench.py --impl reference > $O/${TAG}_bench_ref.json 2> $O/${TAG}_bench_ref.err; echo bench_ref=$?
for c in C3 C4; do
  python bench.py --config $c --no-secondary --no-cpu-baseline > $O/${TAG}_bench_$c.json 2> $O/${TAG}_bench_$c.err; echo bench_$c=$?
done
python tools/full_2p50.py > $O/${TAG}_full_2p50.json 2> $O/${TAG}_full_2p50.err; echo full=$?
# launch list of the bench command (per-launch device times, cold and serialised)
B="bench.py --steps 1 --warmup 3 --min-warmup-s 0 --no-cpu-baseline --no-secondary --prof-steps 1"
python $B > $O/${TAG}_launch_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv \
      --log-file $O/${TAG}_launches_c5.csv python $B > $O/${TAG}_launch_ncu.log 2>&1; echo launches=$?
# full captures: the fused tile kernel near 2^50, the window scan
W="(1<<50)-(1<<38)+1"  # 2^37 odd slots: exactly one C5 batch
# (SQF2K_DEBUG_PAT13_MIN=0: the window takes C5's p <= 13 wheel
# table, i.e. exactly the kernel every C5 batch runs)
export SQF2K_DEBUG_PAT13_MIN=0
python tools/exp_time.py - "$W" "1<<50" > $O/${TAG}_plain_tile.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:tile_kernel -s 2 -c 1 \
      -o $O/${TAG}_prof_tile_c5 python tools/exp_time.py - "$W" "1<<50" > $O/${TAG}_ncu_tile.log 2>&1; echo ncu_tile=$?
unset SQF2K_DEBUG_PAT13_MIN
PIPELINE=bitmap python tools/exp_time.py - "(1<<50)-(1<<37)+1" "1<<50" > $O/${TAG}_plain_scan.log 2>&1 && \
  PIPELINE=bitmap ncu --set full --clock-control none --import-source on -k regex:wscan -s 2 -c 1 \
      -o $O/${TAG}_prof_wscan python tools/exp_time.py - "(1<<50)-(1<<37)+1" "1<<50" > $O/${TAG}_ncu_scan.log 2>&1; echo ncu_scan=$?
