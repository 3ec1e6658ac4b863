mkdir -p gpurun_out
O=gpurun_out/final_check.txt
: > $O
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_all2.log 2>&1
tail -2 gpurun_out/gpu_all2.log >> $O
timeout 600 python tools/dbg_c3flow.py 2>&1 | tail -4 >> $O
EXTRA=200 timeout 600 python tools/dbg_engine.py 2>&1 | tail -4 >> $O
python -c "import __graft_entry__ as g; g.smoke()" >> $O 2>&1; echo "smoke rc=$?" >> $O
cat $O
