export DMF_WATCHDOG_S=20
for cfg in "DMF_ASYNC=0" "DMF_ASYNC_WARPS=8" "DMF_ASYNC_WARPS=12"; do
  echo "## $cfg"; env $cfg timeout 120 python tools/trace_pp.py 20 > gpurun_out/t.txt 2>&1; grep "==" gpurun_out/t.txt | head -4 | tr '\n' ' '; echo
  awk '/== pp/{c++} c==2' gpurun_out/t.txt | grep discharge | cut -c1-150 | head -3
done
