"""ncu target for the roofline's traffic: bench.py's device-resident protocol (handle A:
static solve, warm-up batches with the S_min query, then timed step 0) with the CUDA
profiler switched on only around timed step 0's dmf_apply_batch -- run under
  ncu --profile-from-start off --set full ... python tools/prof_step.py rmat22
Prints that launch's algorithmic bytes (bench.algorithmic_bytes) and device time."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as W
import paper_2511_05895_b200 as P
import bench

wl = sys.argv[1] if len(sys.argv) > 1 else "rmat22"
spec = bench.workload_spec(wl, bench.DEFAULT_WARMUP, bench.DEFAULT_STEPS)
g, batches = W.sequence(spec)
dev = torch.device("cuda", 0)
dbat = [(torch.from_numpy(b.u).to(dev), torch.from_numpy(b.v).to(dev), torch.from_numpy(b.new_cap).to(dev))
        for b in batches]
mask = torch.empty(g.n, dtype=torch.uint8, device=dev)
f = P.DynMaxFlow.from_graph(g)
f.static_solve()
for j in range(bench.DEFAULT_WARMUP):
    f.apply_batch(*dbat[j], algo="pp")
    f.min_cut_source_side(mask)
torch.cuda.synchronize()
torch.cuda.profiler.start()
f.apply_batch(*dbat[bench.DEFAULT_WARMUP], algo="pp")
torch.cuda.synchronize()
torch.cuda.profiler.stop()
st = f.stats()
out = {"workload": wl, "step": "timed step 0 (batch index %d)" % bench.DEFAULT_WARMUP,
       "algorithmic_bytes": bench.algorithmic_bytes(st, g.n), "device_ms": st["device_ms"],
       "certified": st["certified"], "discharge_vertices": st["discharge_vertices"]}
print("STEP", json.dumps(out))
