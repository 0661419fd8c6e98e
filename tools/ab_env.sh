# A/B of runtime knobs on one box: bench.py per setting (argument list of VAR=VALUE sets)
for cfg in "$@"; do
  env $cfg timeout 300 python bench.py --no-cpu-baseline --static-reps 1 > gpurun_out/abenv.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/abenv.json'))
print('$cfg', round(d['ms_per_step'],3), round(d['batch_apply_ms_median'],3), round(d['static_solve_ms_median'],2), {k: round(v) for k, v in d['phase_us_median'].items()})"
done
