#!/bin/bash
# A/B the K3 variants given as library names under build/ab/ (interleaved runs):
# c1 step timing, c3 K3 timing, c4 query join.
cd "$(dirname "$0")/.."
for rep in 1 2; do
for l in "$@"; do
  echo "== $l"
  REFSIG_GPU_LIB=$PWD/build/ab/lib_$l.so python tools/step_timing.py --steps 30 2>&1 | tail -2
  REFSIG_GPU_LIB=$PWD/build/ab/lib_$l.so python tools/k3_timing.py --config c3 --paths tensor --reps 2 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 tiles', round(d['tiles_ms'],3), 'emit', round(d['emit_ms'],3), 'TF', round(d['executed_tflops']))"
done
done
