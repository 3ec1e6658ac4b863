mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:consume_kernel -s 8 -c 1 -o gpurun_out/prof_rowsel -f \
  python tools/tune_sweep.py --layers 4 --steps 2 --grid consume=0 --grid select_rows=1 > gpurun_out/prof_rowsel_run.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:consume_kernel -s 8 -c 1 -o gpurun_out/prof_rowsel_c3 -f \
  python tools/tune_sweep.py --layers 4 --steps 2 --batch 32 --kv 8 --s 16384 --grid consume=0 --grid select_rows=1 > gpurun_out/prof_rowsel_c3_run.log 2>&1
ls -la gpurun_out/*.ncu-rep
