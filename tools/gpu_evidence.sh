# r02 evidence runs (after the split-recall dataflow): profiles, C5, C4, engine step
mkdir -p gpurun_out
bash tools/prof_round.sh > gpurun_out/prof_round.log 2>&1
timeout 1500 python tools/c5_crossover.py --out gpurun_out/r02_c5_crossover.json > gpurun_out/ev_c5.log 2>&1
timeout 1500 python tools/c4_batch_sweep.py --out gpurun_out/r02_c4_batch_sweep.json > gpurun_out/ev_c4.log 2>&1
timeout 900 python tools/engine_step_bench.py --groups 1 --graph 0,1 --out gpurun_out/r02_engine_step.json > gpurun_out/ev_engine.log 2>&1
tail -n 3 gpurun_out/ev_c4.log gpurun_out/ev_engine.log
