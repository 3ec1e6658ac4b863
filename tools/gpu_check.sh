# round check: GPU tests, smoke, C2/C3 bench lines, the reference arm
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/chk_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/chk_pytest.log
tail -n 3 gpurun_out/chk_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/chk_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/chk_smoke.log
tail -n 2 gpurun_out/chk_smoke.log
timeout 500 python bench.py > gpurun_out/chk_c2.log 2>&1
timeout 500 python bench.py --config c3 > gpurun_out/chk_c3.log 2>&1
timeout 500 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/chk_ref.log 2>&1
for f in chk_c2 chk_c3 chk_ref; do python -c "
import json
for l in open('gpurun_out/$f.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$f', round(d['value'],2), round(d['ms_per_step'],3), 'engine', d.get('engine_ms_per_step'), 'e2e', d.get('e2e',{}).get('value'), 'full', d.get('full_kv',{}).get('value'), 'frac', d.get('roofline',{}).get('frac'), 'cpu', d.get('cpu_baseline',{}).get('value'), d.get('clocks'))
"; done
