"""Debug helper: static solve + a few batches on RMAT-`scale`, printing the counters."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import workloads as W
import paper_2511_05895_b200 as P

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 12
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 0
keys = ("iterations", "rounds", "budget_stops", "bfs_levels", "bfs_slots", "discharge_vertices", "discharge_slots",
        "pushes", "relabels", "activations", "stage2_vertices", "bottom_up_levels", "device_ms", "t_prologue_us", "t_reset_us", "t_bfs_us", "t_discharge_us", "t_rie_us", "t_epilogue_us")
g = W.rmat(scale, 16, 1, 7)
f = P.DynMaxFlow.from_graph(g, max_iters=iters)
F = f.static_solve()
st = f.stats()
print("static F", F, {k: st[k] for k in keys}, flush=True)
cs = W.CapState(g)
for j in range(3):
    for algo in ("pp", "pr"):
        b = W.rmat_batch(g, cs, 0.01, 100 + 2 * j + (algo == "pr"))
        cs.apply(b)
        F = f.apply_batch(b.u, b.v, b.new_cap, algo=algo)
        st = f.stats()
        print(algo, "F", F, {k: st[k] for k in keys}, flush=True)
F = f.static_solve(); st = f.stats()
print("re-static F", F, {k: st[k] for k in keys}, flush=True)
