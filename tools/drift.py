"""Per-batch device time and work over a long cumulative DYN_PP sequence on RMAT-20."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import workloads as W
import paper_2511_05895_b200 as P
nb = int(sys.argv[1]) if len(sys.argv) > 1 else 45
g = W.rmat(20, 16, 1, 7)
f = P.DynMaxFlow.from_graph(g)
f.static_solve()
st = W.CapState(g)
for j in range(nb):
    b = W.rmat_batch(g, st, 0.01, 100 + j)
    st.apply(b)
    F = f.apply_batch(b.u, b.v, b.new_cap, algo="pp")
    s = f.stats()
    if j % 3 == 0 or j == nb - 1:
        L = f.export_labels(); e = f.export_state()["e"]
        sexc = int(((L["part"] == 1) & (e > 0)).sum()); tdef = int(((L["part"] == 2) & (e < 0)).sum())
        print(f"b{j:2d} F={F} ms={s['device_ms']:.3f} it={s['iterations']} lv={s['bfs_levels']} bfs_slots={s['bfs_slots']} "
              f"dis_v={s['discharge_vertices']} bfs_us={s['t_bfs_us']:.0f} dis_us={s['t_discharge_us']:.0f} "
              f"S_excess={sexc} T_deficit={tdef} s2={s['stage2_vertices']}", flush=True)
