mkdir -p gpurun_out
O=gpurun_out/chunk1024.txt
: > $O
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_all3.log 2>&1
tail -2 gpurun_out/gpu_all3.log >> $O
timeout 600 python tools/dbg_c3flow.py 2>&1 | tail -4 >> $O
python bench.py --config c3 > gpurun_out/bench_c3b.json 2>/dev/null
python bench.py > gpurun_out/bench_c2b.json 2>/dev/null
for f in bench_c3b bench_c2b; do grep '^{' gpurun_out/$f.json | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print('$f', round(d['value'],1), round(d['ms_per_step'],3), round(d['e2e']['value'],1), round(d['engine_ms_per_step'],3), round(d['roofline']['frac'],3), d['clocks'])" >> $O; done
cat $O
