mkdir -p gpurun_out
O=gpurun_out/flow_sweep7.txt
: > $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_engine_step.py -x -q -p no:cacheprovider > gpurun_out/g7_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/g7_pytest.log
tail -2 gpurun_out/g7_pytest.log >> $O
C2="--layers 16 --steps 10"
echo "== $C2" >> $O
timeout 600 python tools/tune_sweep.py $C2 --grid consume=0 --grid select_rows=0 --profile >> $O 2>&1
timeout 600 python tools/tune_sweep.py $C2 --grid consume=1 --grid consume_gmax=0,1 --grid consume_ctas=48,64 --profile >> $O 2>&1
for i in 1 2; do
timeout 600 python tools/tune_sweep.py $C2 --grid consume=1 --grid consume_gmax=0,1 --grid consume_ctas=40,48,64 >> $O 2>&1
timeout 600 python tools/tune_sweep.py $C2 --engine --grid consume=1 --grid consume_gmax=0,1 --grid consume_ctas=40,48,64 >> $O 2>&1
done
timeout 600 python tools/tune_sweep.py $C2 --engine --grid consume=0 --grid select_rows=0 >> $O 2>&1
timeout 300 python tools/consume_probe.py --tune consume_ctas=48 >> $O 2>&1
timeout 300 python tools/consume_probe.py --tune consume_ctas=48 --engine >> $O 2>&1
cat $O
