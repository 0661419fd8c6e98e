# One GPU call: the bench line, the ncu launch list of a short bench run, and one
# `ncu --set full` capture each of a warm Dynamic Push-Pull batch launch and of the
# static solve launch (RMAT-20).  Outputs land in gpurun_out/ (copied to profiles/).
set -x
timeout 400 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve --launch-skip 2 -c 1 \
  -o gpurun_out/k_solve_pp -f python tools/prof_pp.py pp > gpurun_out/ncu_pp.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve --launch-skip 0 -c 1 \
  -o gpurun_out/k_solve_static -f python tools/prof_pp.py pp > gpurun_out/ncu_static.log 2>&1
