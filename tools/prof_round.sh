#!/bin/bash
# Profiling pass for profiles/: launch list of the bench command, then one
# ncu --set full capture per hot kernel (1 GPU, never multi-rank).
#   bash tools/prof_round.sh ; python tools/summarize_ncu.py <tag>
# gpurun copies back at most 64 MiB of gpurun_out/: select parts with
#   LAUNCHES=0|1  KERNELS="score_fast select_reg recall_pv"  EXTRA="full cand"
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-full-kv"
if [ "${LAUNCHES:-1}" = 1 ]; then
ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 300 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/launches_run.log 2>&1
fi
for k in ${KERNELS-score_fast select_reg recall_pv}; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 200 -c 1 \
      -o gpurun_out/prof_$k -f $CMD > gpurun_out/prof_${k}_run.log 2>&1
done
EXTRA=${EXTRA-full cand}
# the full-KV comparator's fused kernel (bench's full_kv leg)
[[ " $EXTRA " == *" full "* ]] && ncu --set full --clock-control none --import-source on -k regex:full_fast -s 40 -c 1 \
    -o gpurun_out/prof_full_fast -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
    > gpurun_out/prof_full_fast_run.log 2>&1
# candidate mode (auto beyond 32k positions): scoring epilogue + candidate selection at 64k
[[ " $EXTRA " == *" cand "* ]] && ncu --set full --clock-control none --import-source on -k regex:"score_fast|select_cand" -s 6 -c 2 \
    -o gpurun_out/prof_cand64k -f python tools/c5_crossover.py --contexts 65536 --topns 128 --layers 2 --steps 2 \
    > gpurun_out/prof_cand64k_run.log 2>&1
ls -la gpurun_out
