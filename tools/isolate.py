"""Isolate a parity failure: RMAT-`scale` static solve (+ batches) under knob sets, vs Dinic + checker."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
import workloads as W
import paper_2511_05895_b200 as P

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 12
g = W.rmat(scale, 16, 1, 7)
r = O.maxflow(g, "dinic")
sets = {"default": {}, "topo_off": dict(topo_div=-1), "gap_off": dict(local_gap=-1),
        "both_off": dict(topo_div=-1, local_gap=-1), "topology": dict(schedule="topology"),
        "topology_nogap": dict(schedule="topology", local_gap=-1), "async": dict(schedule="async"),
        "rounds": dict(schedule="rounds", topo_div=-1)}
for name, kn in sets.items():
    bad = 0
    for rep in range(3):
        f = P.DynMaxFlow.from_graph(g, **kn)
        F = f.static_solve()
        st = f.export_state()
        smin = f.min_cut_source_side()
        rc, msg, _ = O.check_state(g.n, g.s, g.t, st["row_ptr"], st["dst"], st["rev"], st["cap"], st["res"], st["e"], F, smin)
        s = f.stats()
        ok = F == r["F"] and np.array_equal(smin, r["smin"]) and rc == 0
        bad += not ok
        print(f"{name:16s} rep{rep} F={F} want={r['F']} ok={ok} rc={rc} {msg[:80]} topo_rounds={s['topology_rounds']} gap={s['gap_levels']}/{s['gap_skips']} iters={s['iterations']}")
        f.close()
