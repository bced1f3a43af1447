#!/bin/bash
# Build the protocol-checking variant of the library (-DSQF2K_CHECKS: ring
# ownership tags, barrier-phase and bounds assertions on the device; the
# in-house substitute for compute-sanitizer, which this GPU pool does not
# allow) and run every kernel of the hot path through it on small ranges.
#   bash tools/checks.sh            (build here, run on the box)
cd "$(dirname "$0")/.."
if [ "$1" != "run" ]; then
  bash tools/build_exp.sh "checks=-DSQF2K_CHECKS" && echo built experiments/lib_exp_checks.so
  exit
fi
SQF2K_LIB=$PWD/experiments/lib_exp_checks.so python tools/sanitize.py
