mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/g2_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/g2_pytest.log
timeout 400 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/g2_c2.log 2>&1
timeout 400 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --config c3 > gpurun_out/g2_c3.log 2>&1
timeout 400 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-full-kv --tune consume=0 > gpurun_out/g2_c2_old.log 2>&1
tail -3 gpurun_out/g2_pytest.log
