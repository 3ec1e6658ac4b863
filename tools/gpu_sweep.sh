mkdir -p gpurun_out
O=gpurun_out/sweep_gqa_split.txt
: > $O
C3="--layers 16 --steps 10 --batch 32 --kv 8 --s 16384"
timeout 600 python tools/tune_sweep.py $C3 --grid consume=0 >> $O 2>&1
timeout 600 python tools/tune_sweep.py $C3 --grid consume=2 --grid consume_recall=0 --grid consume_ctas=32,48,64,96 --grid flow_recall_ctas=24,32 >> $O 2>&1
cat $O
