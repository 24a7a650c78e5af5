#!/bin/bash
# Full ncu sections of two K1 kernels for library variants under build/ab/:
#   tools/ncu_k1_full.sh old pack  -> gpurun_out/k1full_<name>.ncu-rep
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for l in "$@"; do
  REFSIG_GPU_LIB=$PWD/build/ab/lib_$l.so timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:count_warp_kernel<\(int\)8>|group_sort_kernel<\(int\)4, \(int\)8>" -c 4 -f -o gpurun_out/k1full_$l \
    python tools/step_timing.py --steps 2 > gpurun_out/k1full_$l.log 2>&1
  tail -2 gpurun_out/k1full_$l.log
done
