"""ncu target: bench.py's protocol (static solve, warm-up batches with the S_min query,
then timed step 0's dmf_apply_batch) with the CUDA profiler on only around timed step
0's dmf_min_cut_source_side (the MINCUT launch) -- run under
  ncu --profile-from-start off --set full ... python tools/prof_cut.py rmat22"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as W
import paper_2511_05895_b200 as P
import bench

wl = sys.argv[1] if len(sys.argv) > 1 else "rmat22"
spec = bench.workload_spec(wl, bench.DEFAULT_WARMUP, 1)
g, batches = W.sequence(spec)
dev = torch.device("cuda", 0)
mask = torch.empty(g.n, dtype=torch.uint8, device=dev)
f = P.DynMaxFlow.from_graph(g)
f.static_solve()
for j, b in enumerate(batches):
    f.apply_batch(b.u, b.v, b.new_cap, algo="pp")
    torch.cuda.synchronize()
    if j == bench.DEFAULT_WARMUP:
        torch.cuda.profiler.start()
    f.min_cut_source_side(mask)
    torch.cuda.synchronize()
    if j == bench.DEFAULT_WARMUP:
        torch.cuda.profiler.stop()
print("CUT", f.stats()["device_ms"])
