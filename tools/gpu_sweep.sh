mkdir -p gpurun_out
O=gpurun_out/sweep_mma3.txt
: > $O
C3="--layers 16 --steps 10 --batch 32 --kv 8 --s 16384"
timeout 600 python tools/tune_sweep.py $C3 --grid score_chunk=0,1024,2048 --profile >> $O 2>&1
timeout 600 python tools/tune_sweep.py $C3 --grid recall_ctas=16,32 >> $O 2>&1
timeout 600 python tools/tune_sweep.py $C3 --engine --grid score_chunk=0 >> $O 2>&1
timeout 600 python tools/kbench.py --help > /dev/null 2>&1
cat $O
