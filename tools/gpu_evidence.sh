# r02 evidence runs: C5 crossover, C4 batch sweep, engine step, prefill offload
mkdir -p gpurun_out
timeout 1500 python tools/c5_crossover.py --out gpurun_out/r02_c5_crossover.json > gpurun_out/ev_c5.log 2>&1
timeout 900 python tools/engine_step_bench.py --groups 1 --graph 0,1 --out gpurun_out/r02_engine_step.json > gpurun_out/ev_engine.log 2>&1
timeout 900 python tools/engine_step_bench.py --groups 1,2 --tune consume=0 --out gpurun_out/r02_engine_step_stream_ordered.json > gpurun_out/ev_engine0.log 2>&1
timeout 900 python tools/prefill_offload_bench.py --out gpurun_out/r02_prefill_offload.json > gpurun_out/ev_prefill.log 2>&1
timeout 1500 python tools/c4_batch_sweep.py --out gpurun_out/r02_c4_batch_sweep.json > gpurun_out/ev_c4.log 2>&1
tail -3 gpurun_out/ev_*.log
