mkdir -p gpurun_out
O=gpurun_out/sweep_nlayers.txt
: > $O
for L in 2 4 8 16 32; do
timeout 600 python tools/tune_sweep.py --layers $L --steps 10 --grid consume_recall=0,1 --grid consume_ctas=0 >> $O 2>&1
done
timeout 600 python tools/tune_sweep.py --layers 8 --steps 10 --s 16384 --grid consume_recall=0,1 >> $O 2>&1
timeout 600 python tools/tune_sweep.py --layers 16 --steps 10 --s 16384 --grid consume_recall=0,1 >> $O 2>&1
cat $O
