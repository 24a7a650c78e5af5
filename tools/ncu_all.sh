#!/bin/bash
# Per-kernel ncu evidence (run on the GPU box, after tools/prof_all.py exited 0 there):
# --set full captures of every kernel at c1 / c3 / c4 reduced ON THE BOX to raw-metric CSVs and
# opcode mixes (the .ncu-rep files are too large to bring back), plus the launch list of the step.
cd "$(dirname "$0")/.."
out=gpurun_out
python tools/step_timing.py --steps 3 > $out/plain_st.log 2>&1 && \
  ncu -f --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_r02.csv \
      python tools/step_timing.py --steps 3 > $out/ncu_l.log 2>&1
for c in c1 c3 c4; do
  set -- $c
  ncu -f --set full --clock-control none --import-source on --nvtx --nvtx-include "measured/" -o /tmp/prof_$1 \
      python tools/prof_all.py --config $1 > $out/ncu_$1.log 2>&1
  ncu -i /tmp/prof_$1.ncu-rep --page raw --csv > $out/ncu_raw_$1.csv 2>/dev/null
  python tools/sass_mix.py /tmp/prof_$1.ncu-rep --top 12 > $out/ncu_mix_$1.txt 2>/dev/null
done
ls -la $out
