for t in "consume=1" "consume=0" "consume=1" "consume=0"; do
python bench.py --config c3 --steps 10 --no-cpu-baseline --no-e2e --no-full-kv --tune $t 2>/dev/null | grep '^{' | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print('c3 $t', round(d['value'],1), round(d['engine_ms_per_step'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
B=32 S=16384 CTAS=48,56,64 EXTRA=300 timeout 600 python tools/dbg_engine.py 2>&1 | tail -4
