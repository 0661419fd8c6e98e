# long cumulative DYN_PP sequences (tools/drift.py) under settings given as "VAR=V VAR2=W" strings
for cfg in "$@"; do
  env $cfg timeout 300 python tools/drift.py 45 > gpurun_out/d.txt 2>&1
  python - "$cfg" <<'PY'
import re, sys
ms = [float(m.group(1)) for m in re.finditer(r"ms=([0-9.]+)", open("gpurun_out/d.txt").read())]
its = re.findall(r"it=(\d+)", open("gpurun_out/d.txt").read())
print(sys.argv[1], "mean %.3f median %.3f max %.3f" % (sum(ms) / len(ms), sorted(ms)[len(ms) // 2], max(ms)), "iters", "".join(its))
PY
done
