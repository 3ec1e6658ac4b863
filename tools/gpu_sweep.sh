mkdir -p gpurun_out
O=gpurun_out/sweep_tma2.txt
: > $O
C3="--layers 16 --steps 10 --batch 32 --kv 8 --s 16384"
nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.active --format=csv,noheader,nounits -lms 100 > gpurun_out/smi_tma2.txt &
SMI=$!
for i in 1 2 3; do
timeout 600 python tools/tune_sweep.py --layers 16 --steps 10 --grid recall_tma=0,1 --grid flow_recall_ctas=16,24 >> $O 2>&1
timeout 600 python tools/tune_sweep.py $C3 --grid recall_tma=0,1 >> $O 2>&1
timeout 600 python tools/tune_sweep.py $C3 --grid recall_tma=0,1 --engine >> $O 2>&1
timeout 600 python tools/tune_sweep.py --layers 16 --steps 10 --grid recall_tma=0,1 --engine >> $O 2>&1
done
kill $SMI
cat $O
