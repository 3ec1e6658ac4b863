mkdir -p gpurun_out
O=gpurun_out/c2recall.txt
: > $O
C2="--layers 16 --steps 10"
timeout 900 python tools/tune_sweep.py $C2 --grid recall_pipe=-1,1 --grid recall_lean=0,1 --grid flow_recall_ctas=16,24 >> $O 2>&1
timeout 900 python tools/tune_sweep.py $C2 --grid recall_pipe=1 --grid recall_dbg=0,1,2 >> $O 2>&1
timeout 900 python tools/tune_sweep.py $C2 --grid recall_tma=1 --grid flow_recall_ctas=16,24 >> $O 2>&1
timeout 900 python tools/tune_sweep.py $C2 --grid pipeline=0 --profile >> $O 2>&1
cat $O
