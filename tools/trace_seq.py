"""Replay the bench sequence (RMAT-20, cumulative 1% batches) and print the phase
trace of selected batches."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W
import paper_2511_05895_b200 as P

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 12
algo = sys.argv[2] if len(sys.argv) > 2 else "pp"
show_from = int(sys.argv[3]) if len(sys.argv) > 3 else nb - 2
g = W.rmat(20, 16, 1, 7)
f = P.DynMaxFlow.from_graph(g)
f.set_trace(8192)
f.static_solve()
st = W.CapState(g)
for j in range(nb):
    b = W.rmat_batch(g, st, 0.01, 100 + j); st.apply(b)
    f.apply_batch(b.u, b.v, b.new_cap, algo=algo)
    s = f.stats()
    ph = {k: round(s[k]) for k in ("t_prologue_us", "t_reset_us", "t_bfs_us", "t_discharge_us", "t_rie_us", "t_epilogue_us")}
    print(f"batch {j}: {s['device_ms']:.3f} ms rounds={s['rounds']} iters={s['iterations']} levels={s['bfs_levels']} {ph}", flush=True)
    if j >= show_from:
        for r in f.trace():
            ex = r['extra']
            extra = f"bu={ex & 3} sp={(ex >> 2) & 1} ch={ex >> 3}" if r['phase'] == 'bfs' else f"x={ex}"
            sl = f"  slowest {r['slow_us']:.1f}us deg={r['slow_deg']} cyc={r['slow_cyc']}" if r['phase'] == 'discharge' else ""
            print(f"  {r['phase']:9s} it={r['iter']:<3d} sub={r['sub']:<4d} items={r['items']:<9d} {extra:18s} {r['us']:9.1f} us{sl}")
