"""Print the per-phase trace of PP batches (bench sequence) / a PR batch / static solve on RMAT.
usage: python tools/trace_pp.py [scale] [skip] [show]   -- skip untraced PP batches first, then trace `show`"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import workloads as W
import paper_2511_05895_b200 as P

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
nshow = int(sys.argv[3]) if len(sys.argv) > 3 else 2
g = W.rmat(scale, 16, 1, 7)
f = P.DynMaxFlow.from_graph(g)
f.set_trace(8192)
def show(tag):
    st = f.stats()
    print(f"== {tag}: {st['device_ms']:.3f} ms  iters={st['iterations']} levels={st['bfs_levels']} bfs_slots={st['bfs_slots']} "
          f"bfs_v={st['bfs_vertices']} dis_v={st['discharge_vertices']} pushes={st['pushes']} s2={st['stage2_vertices']}")
    cta = f.trace_cta()
    for ri, r in enumerate(f.trace()):
        ex = r['extra']
        extra = f"bu={ex & 3} ch={ex >> 3}" if r['phase'] == 'bfs' else f"x={ex}"
        if r['phase'] == 'bfs' and r['slow_us'] > 0:
            extra += f" slowchunk={r['slow_us']:.1f}us v={(int(r['slow_deg']) << 8) | int(r['slow_cyc'])}"
        if r['phase'] == 'discharge':
            extra += f" slow={r['slow_us']:.1f}us deg={r['slow_deg']} cyc={r['slow_cyc']}"
        c = np.sort(cta[ri]) if ri < len(cta) else np.zeros(1)
        dist = f"cta busy p50={c[len(c) // 2]:.1f} p90={c[int(len(c) * .9)]:.1f} max={c[-1]:.1f}"
        if ri < len(cta) and len(cta[ri]):
            dist += f" (cta {int(np.argmax(cta[ri]))})"
        print(f"  {r['phase']:9s} it={r['iter']:<3d} sub={r['sub']:<4d} items={r['items']:<9d} {extra:16s} {r['us']:9.1f} us  {dist}")
f.static_solve_pp(); show("static_pp")
f.static_solve(); show("static")
cs = W.CapState(g)
for j in range(skip + nshow):
    b = W.rmat_batch(g, cs, 0.01, 100 + j); cs.apply(b)
    f.apply_batch(b.u, b.v, b.new_cap, algo="pp")
    if j >= skip:
        show(f"pp batch {j}")
m = f.min_cut_source_side(); show("mincut (cached)")
b = W.rmat_batch(g, cs, 0.01, 100 + skip + nshow); cs.apply(b)
f.apply_batch(b.u, b.v, b.new_cap, algo="pr"); show("pr")
m = f.max_cut_source_side(); show("maxcut")
