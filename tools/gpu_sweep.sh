mkdir -p gpurun_out
O=gpurun_out/pinfirst.txt
: > $O
for i in 1 2; do
python bench.py --no-cpu-baseline --no-full-kv > gpurun_out/pf_c2_$i.json 2>gpurun_out/pf_c2_$i.err
grep '^{' gpurun_out/pf_c2_$i.json | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print('c2', round(d['value'],1), round(d['ms_per_step'],3), round(d['e2e']['value'],1), round(d['engine_ms_per_step'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> $O
cat gpurun_out/pf_c2_$i.err >> $O
done
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_all4.log 2>&1
tail -2 gpurun_out/gpu_all4.log >> $O
cat $O
