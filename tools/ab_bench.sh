# A/B on one box: bench.py with HEAD in rounds mode vs asynchronous mode
for v in async; do
  if [ $v = sync ]; then export DMF_ASYNC=0; else unset DMF_ASYNC; fi
  timeout 300 python bench.py --no-cpu-baseline > gpurun_out/ab_$v.json 2>> gpurun_out/ab.err
done
