# round check: GPU tests, smoke, C2/C3 bench lines (and optional evidence tools)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/chk_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/chk_pytest.log
tail -n 3 gpurun_out/chk_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/chk_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/chk_smoke.log
tail -n 2 gpurun_out/chk_smoke.log
timeout 500 python bench.py > gpurun_out/chk_c2.log 2>&1
timeout 500 python bench.py --config c3 > gpurun_out/chk_c3.log 2>&1
for f in chk_c2 chk_c3; do python -c "
import json
for l in open('gpurun_out/$f.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$f', round(d['value'],1), round(d['ms_per_step'],3), 'engine', d.get('engine_ms_per_step'), 'e2e', d.get('e2e',{}).get('value'), 'full', d.get('full_kv',{}).get('value'), 'frac', d.get('roofline',{}).get('frac'), d.get('clocks'))
"; done
if [ -n "$EVIDENCE" ]; then
timeout 900 python tools/engine_step_bench.py --groups 1 --graph 0,1 --out gpurun_out/r02_engine_step.json > gpurun_out/ev_engine.log 2>&1
timeout 900 python tools/prefill_offload_bench.py --out gpurun_out/r02_prefill_offload.json > gpurun_out/ev_prefill.log 2>&1
tail -n 2 gpurun_out/ev_engine.log gpurun_out/ev_prefill.log
fi
