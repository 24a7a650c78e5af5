#!/bin/bash
# A/B K2 variants given as library names under build/ab/ (interleaved runs):
# c3 sign timing (cold L2) and the c1 step.
cd "$(dirname "$0")/.."
for rep in 1 2; do
for l in "$@"; do
  echo "== $l"
  REFSIG_GPU_LIB=$PWD/build/ab/lib_$l.so python tools/sign_timing.py --config c3 --reps 10 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 sign ms', round(d['ms'],4), 'frac', round(d['frac'],3))"
  REFSIG_GPU_LIB=$PWD/build/ab/lib_$l.so python tools/sign_timing.py --config c1 --reps 20 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1 sign ms', round(d['ms'],4), 'frac', round(d['frac'],3))"
  REFSIG_GPU_LIB=$PWD/build/ab/lib_$l.so python tools/step_timing.py --steps 30 2>&1 | tail -2
done
done
