mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "prefill or staged" > gpurun_out/pf_pytest.log 2>&1; tail -n 2 gpurun_out/pf_pytest.log
timeout 900 python tools/prefill_offload_bench.py --out gpurun_out/r02_prefill_offload.json > gpurun_out/ev_prefill.log 2>&1
python -c "
import json; d=json.load(open('gpurun_out/r02_prefill_offload.json')); print(d['staged_offload_gbs'], {k:v['total_ms'] for k,v in d['timelines'].items()}, d['offload_cost_ms'])"
