# A/B of alternative builds (abtmp/libdmf_*.so) against the in-tree library, one box
P=paper_2511_05895_b200
cp $P/libdmf.so /tmp/libdmf_cur.so
for v in cur "$@"; do
  if [ $v = cur ]; then cp /tmp/libdmf_cur.so $P/libdmf.so; else cp abtmp/libdmf_$v.so $P/libdmf.so; fi
  timeout 300 python bench.py --no-cpu-baseline --static-reps 2 > gpurun_out/ablib.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ablib.json'))
print('$v', round(d['ms_per_step'],3), round(d['batch_apply_ms_median'],3), round(d['static_solve_ms_median'],2), {k: round(v) for k, v in d['phase_us_median'].items()})"
done
cp /tmp/libdmf_cur.so $P/libdmf.so
