#!/bin/bash
# Profiling pass for profiles/ (1 GPU, never multi-rank): the launch lists of
# the C2 and C3 bench commands, then one `ncu --set full` capture per hot
# kernel, exported to raw CSV on the box (the .ncu-rep files are large).
#   bash tools/prof_round.sh ; python tools/summarize_ncu.py <tag>
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-full-kv --no-engine"
ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 300 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/launches_run.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -s 400 -c 400 --csv \
    --log-file gpurun_out/launches_c3.csv $CMD --config c3 > gpurun_out/launches_c3_run.log 2>&1
cap() {  # name, kernel regex, skip, extra bench args
  ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 \
      -o gpurun_out/prof_$1 -f $CMD $4 > gpurun_out/prof_$1_run.log 2>&1
  ncu -i gpurun_out/prof_$1.ncu-rep --page raw --csv > gpurun_out/prof_$1_raw.csv 2>/dev/null
}
if [ -z "$ONLY" ]; then
cap score_fast score_fast 200 ""
cap consume consume_kernel 60 ""
cap score_mma_c3 score_mma 200 "--config c3"
cap recall_pv_c3 recall_pv 60 "--config c3"
fi
cap recall_pv recall_pv 60 ""
cap select_cached_c3 select_rows_cached 60 "--config c3"
[ -n "$ONLY" ] && exit 0
# the full-KV comparator's fused kernel (bench's full_kv leg)
ncu --set full --clock-control none --import-source on -k regex:full_fast -s 40 -c 1 \
    -o gpurun_out/prof_full_fast -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-engine \
    > gpurun_out/prof_full_fast_run.log 2>&1
ncu -i gpurun_out/prof_full_fast.ncu-rep --page raw --csv > gpurun_out/prof_full_fast_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_consume.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof_consume_source.csv 2>/dev/null
# keep only the consumer's report (source view); the rest travel as CSV
for f in gpurun_out/prof_*.ncu-rep; do [ "$f" = gpurun_out/prof_consume.ncu-rep ] || rm -f "$f"; done
ls -la gpurun_out
