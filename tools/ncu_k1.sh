#!/bin/bash
# Per-kernel K1 durations (ncu, serialised, cold-ish) for library variants under build/ab/:
#   tools/ncu_k1.sh old pack  -> gpurun_out/k1_<name>.csv
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for l in "$@"; do
  REFSIG_GPU_LIB=$PWD/build/ab/lib_$l.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none \
    -k "regex:count_warp|group_sort|group_split|idf_kernel" --csv --log-file gpurun_out/k1_$l.csv \
    python tools/step_timing.py --steps 3 > /dev/null 2>&1
  python3 - "$l" <<'PY'
import csv, sys, collections
name = sys.argv[1]
rows = [r for r in csv.reader(open(f"gpurun_out/k1_{name}.csv")) if len(r) > 10]
hdr = rows[0]; ki = hdr.index("Kernel Name"); vi = hdr.index("Metric Value"); ui = hdr.index("Metric Unit")
d = collections.defaultdict(list)
for r in rows[1:]:
    v = float(r[vi].replace(",", "")); v = v / 1000 if r[ui] == "nsecond" else v
    d[r[ki].split("(")[0]].append(v)
tot = 0
for k, v in sorted(d.items(), key=lambda x: -sum(x[1]) / len(x[1])):
    v.sort(); med = v[len(v) // 2]; tot += med
    print(f"{name:6s} {k[:48]:48s} n={len(v):3d} med {med:7.2f} us")
print(f"{name:6s} sum of medians {tot:.1f} us")
PY
done
