mkdir -p gpurun_out
timeout 500 python bench.py --dist peaked --no-cpu-baseline --no-full-kv > gpurun_out/peaked_c2.log 2>&1
timeout 500 python bench.py --dist peaked --config c3 --no-cpu-baseline --no-full-kv > gpurun_out/peaked_c3.log 2>&1
for f in peaked_c2 peaked_c3; do python -c "
import json
for l in open('gpurun_out/$f.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$f', round(d['value'],1), round(d['ms_per_step'],3), 'engine', d.get('engine_ms_per_step'), 'e2e', d.get('e2e',{}).get('value'), d['kernel_ms_per_step'])
"; done
tail -n 3 gpurun_out/peaked_c2.log | cut -c1-300
timeout 1500 python tools/c5_crossover.py --out gpurun_out/r02_c5_crossover.json > gpurun_out/ev_c5.log 2>&1
tail -n 2 gpurun_out/ev_c5.log | cut -c1-200
