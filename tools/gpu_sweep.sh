mkdir -p gpurun_out
O=gpurun_out/sweep_cached.txt
: > $O
timeout 900 python -m pytest tests/test_gpu_dataflow.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider -k "cached or c3 or consumer" > gpurun_out/cached_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/cached_pytest.log
tail -n 2 gpurun_out/cached_pytest.log >> $O
C3="--layers 16 --steps 10 --batch 32 --kv 8 --s 16384"
timeout 600 python tools/tune_sweep.py $C3 --grid select_cached=0,1 --profile >> $O 2>&1
timeout 600 python tools/tune_sweep.py $C3 --grid select_cached=0,1 >> $O 2>&1
timeout 600 python tools/tune_sweep.py $C3 --engine --grid select_cached=0,1 >> $O 2>&1
cat $O
