"""Phase trace of bench.py's step (dmf_apply_batch DYN_PP + dmf_min_cut_source_side) on
its own workload: replays the warm-up batches untraced, then prints the per-phase trace
(and per-CTA busy spread) of `show` timed steps, both launches of each.
usage: python tools/trace_step.py [rmat22|rmat20] [show]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import workloads as W
import paper_2511_05895_b200 as P
import bench

wl = sys.argv[1] if len(sys.argv) > 1 else "rmat22"
nshow = int(sys.argv[2]) if len(sys.argv) > 2 else 2
spec = bench.workload_spec(wl, bench.DEFAULT_WARMUP, nshow)
g, batches = W.sequence(spec)
f = P.DynMaxFlow.from_graph(g)


def show(tag):
    st = f.stats()
    print(f"== {tag}: {st['device_ms']:.3f} ms iters={st['iterations']} levels={st['bfs_levels']} "
          f"bfs_v={st['bfs_vertices']} bfs_slots={st['bfs_slots']} dis_v={st['discharge_vertices']} "
          f"dis_slots={st['discharge_slots']} pushes={st['pushes']} relabels={st['relabels']} "
          f"cert={st['certified']} tail={st['tail_stops']} budget={st['budget_stops']}", flush=True)
    cta = f.trace_cta()
    for ri, r in enumerate(f.trace()):
        ex = r['extra']
        extra = f"bu={ex & 3} ch={ex >> 3}" if r['phase'].startswith('bfs') else f"x={ex}"
        c = np.sort(cta[ri]) if ri < len(cta) else np.zeros(1)
        dist = f"cta p50={c[len(c) // 2]:.1f} max={c[-1]:.1f}" if len(c) else ""
        print(f"  {r['phase']:9s} it={r['iter']:<3d} sub={r['sub']:<4d} items={r['items']:<9d} {extra:16s} "
              f"{r['us']:9.1f} us  {dist}")


f.static_solve()
for j, b in enumerate(batches):
    if j == bench.DEFAULT_WARMUP:
        f.set_trace(8192)
    f.apply_batch(b.u, b.v, b.new_cap, algo="pp")
    if j >= bench.DEFAULT_WARMUP:
        show(f"apply batch {j}")
    f.min_cut_source_side()
    if j >= bench.DEFAULT_WARMUP:
        show(f"min cut after batch {j}")
        print("   |S_min| =", int(f.min_cut_source_side().sum()), "of", g.n)
