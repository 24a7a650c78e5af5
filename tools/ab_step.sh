#!/bin/bash
# A/B whole-step timing of library variants under build/ab/ (interleaved runs).
cd "$(dirname "$0")/.."
for rep in 1 2 3; do
for l in "$@"; do
  echo "== $l"
  REFSIG_GPU_LIB=$PWD/build/ab/lib_$l.so python tools/step_timing.py --steps 30 2>&1 | tail -2
done
done
