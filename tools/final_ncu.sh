# ncu evidence at HEAD (after the bench line): launch list of a short bench run and full
# captures of timed step 0's dmf_apply_batch launches and of its S_min query (RMAT-22).
set -x
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --profile-from-start off --set full --metrics lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum \
  --clock-control none --import-source on -k regex:"k_solve|k_reach" -c 3 -o gpurun_out/step0 -f \
  python tools/prof_step.py rmat22 > gpurun_out/ncu_step0.log 2>&1
timeout 900 ncu --profile-from-start off --set full --metrics lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum \
  --clock-control none --import-source on -k regex:k_reach -c 1 -o gpurun_out/cut0 -f \
  python tools/prof_cut.py rmat22 > gpurun_out/ncu_cut0.log 2>&1
echo done
