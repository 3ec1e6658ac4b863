mkdir -p gpurun_out
for i in 1 2 3; do
  timeout 1100 python -m pytest tests -m gpu -x -q -p no:cacheprovider --tb=long > gpurun_out/flaky_$i.log 2>&1
  rc=$?
  tail -2 gpurun_out/flaky_$i.log
  if [ $rc -ne 0 ]; then break; fi
done
