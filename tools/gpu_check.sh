mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/g8_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/g8_pytest.log
tail -3 gpurun_out/g8_pytest.log
timeout 400 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/g8_c2.log 2>&1
timeout 400 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --config c3 > gpurun_out/g8_c3.log 2>&1
for f in g8_c2 g8_c3; do python -c "
import json
for l in open('gpurun_out/$f.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$f', d['value'], d['ms_per_step'], d.get('engine_ms_per_step'), d.get('e2e',{}).get('value'), d.get('full_kv',{}).get('value'), d.get('roofline',{}).get('frac'))
"; done
