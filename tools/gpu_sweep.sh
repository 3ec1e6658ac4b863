mkdir -p gpurun_out
for t in "consume_ctas=0" "consume_ctas=40" "consume_ctas=0" "consume_ctas=40"; do
python bench.py --steps 20 --no-cpu-baseline --no-e2e --no-full-kv --tune $t 2>/dev/null | grep '^{' | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print('c2 $t', round(d['value'],1), round(d['engine_ms_per_step'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
