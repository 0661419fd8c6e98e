"""Launch sequence for ncu, the bench's protocol: static solve (launch 0), then DYN_PP
batches each followed by the S_min query: pp0 (1), cut0 (2), pp1 (3), cut1 (4), pp2 (5) ...
usage: python tools/prof_pp.py [scale] [nbatches] [algo]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W
import paper_2511_05895_b200 as P

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 3
algo = sys.argv[3] if len(sys.argv) > 3 else "pp"
g, batches = W.sequence(dict(kind="rmat", scale=scale, frac=0.01, nb=nb))
f = P.DynMaxFlow.from_graph(g)
f.static_solve()
for b in batches:
    f.apply_batch(b.u, b.v, b.new_cap, algo=algo)
    print("batch ms", f.stats()["device_ms"], flush=True)
    f.min_cut_source_side()
print("done", f.flow_value())
