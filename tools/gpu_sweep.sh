mkdir -p gpurun_out
O=gpurun_out/probe_cached2.txt
: > $O
timeout 300 python tools/consume_probe.py --layers 4 --batch 32 --heads 32 --kv 8 --s 16384 --tune consume=0 >> $O 2>&1
timeout 300 python tools/consume_probe.py --layers 4 --batch 8 --heads 32 --kv 32 --s 32768 >> $O 2>&1
C3="--layers 16 --steps 10 --batch 32 --kv 8 --s 16384"
timeout 600 python tools/tune_sweep.py $C3 --grid select_cached=1 --profile >> $O 2>&1
timeout 600 python tools/tune_sweep.py --layers 16 --steps 10 --grid consume=1 >> $O 2>&1
timeout 600 python -m pytest tests/test_gpu_dataflow.py tests/test_gpu_candidates.py -x -q -p no:cacheprovider >> $O 2>&1
cat $O
