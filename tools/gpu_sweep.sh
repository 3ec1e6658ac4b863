mkdir -p gpurun_out
O=gpurun_out/sweep_split2.txt
: > $O
C2="--layers 16 --steps 10"
for i in 1 2; do
timeout 600 python tools/tune_sweep.py $C2 --grid consume_ctas=28,32,36,40 --grid recall_ctas=16,24,32 >> $O 2>&1
done
timeout 600 python tools/tune_sweep.py $C2 --grid recall_pipe=0,1 --grid recall_ctas=24,32 >> $O 2>&1
cat $O
