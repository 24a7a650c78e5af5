#!/bin/bash
# A/B variant of the library: recompile ONE source file with extra defines and
# link it with the other (current) objects into build/ab/lib_<name>.so.
#   tools/ab_build.sh <name> <source.cu basename, e.g. k3_tc> "<-DFOO=1 ...>"
# AB_REPLACES=<object basename> when the source is a renamed copy (e.g. an old revision).
set -e
cd "$(dirname "$0")/.."
name=$1; src=$2; defs=$3
mkdir -p build/ab
NV=/usr/local/cuda/bin/nvcc
FLAGS="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Iinclude --expt-relaxed-constexpr"
$NV $FLAGS $defs -c paper_1810_03099_b200/csrc/$src.cu -o build/ab/${src}_$name.o
objs=$(ls build/*.o | grep -v "/${AB_REPLACES:-$src}.o")
$NV -gencode arch=compute_100a,code=sm_100a -shared $objs build/ab/${src}_$name.o -o build/ab/lib_$name.so -lcudart
echo build/ab/lib_$name.so
