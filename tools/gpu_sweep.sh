mkdir -p gpurun_out
O=gpurun_out/c2recall20.txt
: > $O
nvidia-smi --query-gpu=clocks.sm,power.draw,power.limit,clocks_event_reasons.active --format=csv,noheader >> $O
for i in 1 2 3; do
timeout 900 python tools/tune_sweep.py --layers 16 --steps 10 --grid flow_recall_ctas=16,20,24 >> $O 2>&1
done
for t in "flow_recall_ctas=20" "flow_recall_ctas=24" "flow_recall_ctas=20" "flow_recall_ctas=24"; do
python bench.py --steps 20 --no-cpu-baseline --no-e2e --no-full-kv --no-engine --tune $t 2>/dev/null | grep '^{' | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print('bench $t', round(d['value'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> $O
done
cat $O
