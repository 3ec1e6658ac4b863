#!/bin/bash
# Profiling pass: isolated-kernel bench (no recall overlap), launch list, ncu --set full of the scoring kernel.
mkdir -p gpurun_out
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --tune pipeline=0 > gpurun_out/bench_nopipe.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 200 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/launches_run.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:score_fast -s 40 -c 1 -o gpurun_out/prof_score -f \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof_score_run.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:select_kernel -s 40 -c 1 -o gpurun_out/prof_select -f \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof_select_run.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:recall_pv -s 40 -c 1 -o gpurun_out/prof_recall -f \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof_recall_run.log 2>&1
tail -c 3000 gpurun_out/bench_nopipe.log
ls -la gpurun_out
