mkdir -p gpurun_out
timeout 900 python tools/c5_crossover.py --contexts 16384,32768,65536 --topns 128,256 --out gpurun_out/c5_check.json > /dev/null 2>&1
python - <<'PY'
import json
new=json.load(open('gpurun_out/c5_check.json')); old=json.load(open('profiles/r02_c5_crossover.json'))
o={(r['s'],r['top_n']):r['per_layer_us'] for r in old['rows']}
for r in new['rows']:
    k=(r['s'],r['top_n']); print(k, round(o[k],1), '->', round(r['per_layer_us'],1))
PY
for t in "flow_recall_ctas=0" "flow_recall_ctas=24" "flow_recall_ctas=0" "flow_recall_ctas=24"; do
python bench.py --steps 20 --no-cpu-baseline --no-e2e --no-full-kv --no-engine --tune $t 2>/dev/null | grep '^{' | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print('bench $t', round(d['value'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
