mkdir -p gpurun_out
O=gpurun_out/gqa_auto2.txt
: > $O
for t in "consume=1" "consume=0" "consume=1" "consume=0"; do
python bench.py --config c3 --steps 10 --no-cpu-baseline --no-full-kv --tune $t 2>/dev/null | grep '^{' | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print('c3 $t', round(d['value'],1), round(d['e2e']['value'],1), round(d['engine_ms_per_step'],3), d['clocks']['sm_mhz'])" >> $O
done
C3="--layers 16 --steps 10 --batch 32 --kv 8 --s 16384"
timeout 900 python tools/tune_sweep.py $C3 --engine --grid consume=0,1 >> $O 2>&1
for shape in "--batch 16 --s 32768" "--batch 8 --s 65536"; do
timeout 900 python tools/tune_sweep.py --layers 8 --steps 8 --kv 8 $shape --engine --grid consume=0,1 >> $O 2>&1
done
cat $O
