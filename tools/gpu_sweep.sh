mkdir -p gpurun_out
O=gpurun_out/sweep_cachedU.txt
: > $O
timeout 600 python -m pytest tests/test_gpu_dataflow.py -x -q -p no:cacheprovider -k "cached or bitwise" > gpurun_out/cu_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/cu_pytest.log
tail -n 2 gpurun_out/cu_pytest.log >> $O
C3="--layers 16 --steps 10 --batch 32 --kv 8 --s 16384"
for i in 1 2; do
timeout 600 python tools/tune_sweep.py $C3 --grid select_cached=0,1 --profile >> $O 2>&1
done
cat $O
