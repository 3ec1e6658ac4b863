mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_candidates.py tests/test_gpu_dataflow.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/t_lean.log 2>&1
tail -3 gpurun_out/t_lean.log
