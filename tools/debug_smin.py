"""Debug: RMAT-20 static + one 1% PP batch; compare S_min with the oracle and dump the differing vertices."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import workloads as W
import oracle as O
import paper_2511_05895_b200 as P
g = W.config_graph("rmat20")
f = P.DynMaxFlow.from_graph(g)
f.static_solve()
st = W.CapState(g)
b = W.rmat_batch(g, st, 0.01, 100)
st.apply(b)
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 1):
    f.apply_batch(b.u, b.v, b.new_cap, algo="pp")
    print("stats", {k: v for k, v in f.stats().items() if not k.startswith('t_')})
    G = st.graph()
    r = O.maxflow(G, "fifo_pr")
    F = f.flow_value(); smin = f.min_cut_source_side(); smax = f.max_cut_source_side()
    print("F", F, r["F"], "smin diff", np.nonzero(smin != r["smin"])[0][:20], "smax diff", np.nonzero(smax != r["smax"])[0][:20])
    L0 = f.export_labels(); print("mirror mismatches", int((L0["rres"] != f.export_state()["res"][f.export_state()["rev"]]).sum()))
    smin2 = f.min_cut_source_side()   # after max_cut: recomputed by a MODE_MINCUT launch
    print("recomputed smin diff", np.nonzero(smin2 != r["smin"])[0][:20])
    L = f.export_labels()
    s = f.export_state()
    rc, msg, _ = O.check_state(G.n, G.s, G.t, s["row_ptr"], s["dst"], s["rev"], s["cap"], s["res"], s["e"], F, smin)
    print("checker", rc, msg)
    for v in np.nonzero(smin != r["smin"])[0][:5]:
        a, z = s["row_ptr"][v], s["row_ptr"][v + 1]
        print("labels", "hp", L["hp"][v], "hm", L["hm"][v], "part", L["part"][v])
        print(f"v={v} e={s['e'][v]} deg={z-a} gpu_smin={smin[v]} or_smin={r['smin'][v]} gpu_smax={smax[v]} or_smax={r['smax'][v]}")
        for i in range(a, min(z, a + 12)):
            w = s["dst"][i]
            print(f"   -> {w} hp={L['hp'][w]} hm={L['hm'][w]} part={L['part'][w]} mirror={L['rres'][i]} res={s['res'][i]} rres={s['res'][s['rev'][i]]} e={s['e'][w]} smin_w={smin[w]}/{r['smin'][w]}")
