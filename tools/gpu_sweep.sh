mkdir -p gpurun_out
O=gpurun_out/gate.txt
: > $O
for t in "flow_gate=1" "flow_gate=0" "flow_gate=1" "flow_gate=0"; do
python bench.py --steps 10 --no-cpu-baseline --no-e2e --no-full-kv --tune $t 2>/dev/null | grep '^{' | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print('c2 $t', round(d['value'],1), round(d['engine_ms_per_step'],3), d['clocks']['sm_mhz'])" >> $O
done
for t in "consume=2" "consume=0"; do
python bench.py --config c3 --steps 10 --no-cpu-baseline --no-e2e --no-full-kv --tune $t 2>/dev/null | grep '^{' | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print('c3 $t', round(d['value'],1), round(d['engine_ms_per_step'],3), d['clocks']['sm_mhz'])" >> $O
done
EXTRA=200 timeout 600 python tools/dbg_engine.py 2>&1 | tail -4 >> $O
cat $O
