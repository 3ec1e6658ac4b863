#!/bin/bash
# Profiling pass for profiles/: launch list of the bench command, then one
# ncu --set full capture per hot kernel (1 GPU, never multi-rank).
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 300 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/launches_run.log 2>&1
for k in score_fast select_reg recall_pv; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 200 -c 1 \
      -o gpurun_out/prof_$k -f $CMD > gpurun_out/prof_${k}_run.log 2>&1
done
ls -la gpurun_out
