mkdir -p gpurun_out
O=gpurun_out/consume_probe.txt
: > $O
for ctas in 32 64; do
timeout 300 python tools/consume_probe.py --tune consume_ctas=$ctas >> $O 2>&1
timeout 300 python tools/consume_probe.py --tune consume_ctas=$ctas --engine >> $O 2>&1
timeout 300 python tools/consume_probe.py --batch 32 --kv 8 --s 16384 --tune consume_ctas=$ctas >> $O 2>&1
timeout 300 python tools/consume_probe.py --batch 32 --kv 8 --s 16384 --tune consume_ctas=$ctas --engine >> $O 2>&1
done
cat $O
