"""Launch sequence for ncu: static solve (launch 1), PP batch (2), PP batch (3, profiled), cut (4)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W
import paper_2511_05895_b200 as P

algo = sys.argv[1] if len(sys.argv) > 1 else "pp"
g = W.rmat(20, 16, 1, 7)
f = P.DynMaxFlow.from_graph(g)
f.static_solve()
cs = W.CapState(g)
for j in range(2):
    b = W.rmat_batch(g, cs, 0.01, 100 + j)
    cs.apply(b)
    f.apply_batch(b.u, b.v, b.new_cap, algo=algo)
f.min_cut_source_side()
print("done", f.flow_value(), f.stats()["device_ms"])
