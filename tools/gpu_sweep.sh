mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_all.log 2>&1
tail -5 gpurun_out/gpu_all.log
