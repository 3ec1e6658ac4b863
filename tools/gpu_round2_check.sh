set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv > gpurun_out/g1_smi.txt
free -g >> gpurun_out/g1_smi.txt; nproc >> gpurun_out/g1_smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/g1_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/g1_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g1_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/g1_smoke.log
timeout 600 python bench.py > gpurun_out/g1_bench_c2.log 2>&1
timeout 600 python bench.py --config c3 > gpurun_out/g1_bench_c3.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/g1_bench_ref.log 2>&1
tail -3 gpurun_out/g1_*.log
