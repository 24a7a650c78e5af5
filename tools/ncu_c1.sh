cd $GRAFT_REPO_ROOT
out=gpurun_out
python tools/step_timing.py --steps 3 > $out/plain_st.log 2>&1 && \
  ncu -f --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_r02.csv \
      python tools/step_timing.py --steps 3 > $out/ncu_l.log 2>&1
python tools/prof_all.py --config c1 > $out/plain_prof_c1.log 2>&1 && \
ncu -f --set full --clock-control none --import-source on --nvtx --nvtx-include "measured/" -o /tmp/prof_c1 \
      python tools/prof_all.py --config c1 > $out/ncu_c1.log 2>&1
ncu -i /tmp/prof_c1.ncu-rep --page raw --csv > $out/ncu_raw_c1.csv 2>/dev/null
python tools/sass_mix.py /tmp/prof_c1.ncu-rep --top 12 > $out/ncu_mix_c1.txt 2>/dev/null
ls -la $out | tail -5
