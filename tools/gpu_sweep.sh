mkdir -p gpurun_out
O=gpurun_out/sweep_recall72.txt
: > $O
C3="--layers 16 --steps 10 --batch 32 --kv 8 --s 16384"
timeout 600 python tools/tune_sweep.py $C3 --grid recall_ctas=32,48,64,96 --profile >> $O 2>&1
timeout 600 python tools/tune_sweep.py $C3 --grid recall_ctas=32,48,64 >> $O 2>&1
timeout 600 python tools/tune_sweep.py $C3 --engine --grid recall_ctas=32,48 >> $O 2>&1
cat $O
