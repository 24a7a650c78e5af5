#!/bin/bash
# A/B K5 variants under build/ab/ (interleaved): exact_pairs / evaluate timing at configs[1].
cd "$(dirname "$0")/.."
for rep in 1 2; do
for l in "$@"; do
  echo "== $l"
  REFSIG_GPU_LIB=$PWD/build/ab/lib_$l.so python tools/exact_timing.py 2>&1 | tail -1
done
done
