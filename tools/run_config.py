"""Run one BASELINE config at full size: static solve + a few batches, timing each
call, optionally verifying F / S_min against the oracle.  Usage:
  python tools/run_config.py rmat20|grid2048|bip4m|rmat22_1 [algo pp|pr] [nbatch] [frac] [verify 0|1]"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import workloads as W
import paper_2511_05895_b200 as P

name = sys.argv[1]
algo = sys.argv[2] if len(sys.argv) > 2 else "pp"
nb = int(sys.argv[3]) if len(sys.argv) > 3 else 3
frac = float(sys.argv[4]) if len(sys.argv) > 4 else 0.01
verify = int(sys.argv[5]) if len(sys.argv) > 5 else 0
t = time.time(); g = W.config_graph(name); tg = time.time() - t
t = time.time(); f = P.DynMaxFlow.from_graph(g); tc = time.time() - t
print(f"{name}: n={g.n} m={g.m} S={f.S} gen {tg:.1f}s create {tc:.1f}s", flush=True)
keys = ("iterations", "rounds", "bfs_levels", "bfs_slots", "discharge_slots", "pushes", "relabels", "device_ms",
        "t_bfs_us", "t_discharge_us", "t_rie_us")
def show(tag, F):
    st = f.stats()
    print(f"  {tag}: F={F} " + " ".join(f"{k}={st[k]:.1f}" if isinstance(st[k], float) else f"{k}={st[k]}" for k in keys), flush=True)
def check(gg, F):
    if not verify:
        return
    import oracle as O
    t = time.time(); r = O.maxflow(gg, "fifo_pr"); to = time.time() - t
    m = f.min_cut_source_side()
    print(f"    oracle F={r['F']} ({to:.1f}s) F_ok={r['F'] == F} smin_ok={np.array_equal(m, r['smin'])}", flush=True)
F = f.static_solve_pp(); show("static-pp", F)
F = f.static_solve(); show("static", F); check(g, F)
st = W.CapState(g)
for j in range(nb):
    if name.startswith("grid"):
        b = W.grid_batch(g, frac, 300 + j)
    elif name.startswith("bip"):
        b = W.bipartite_batch(g, st, frac, 400 + j)
    else:
        b = W.rmat_batch(g, st, frac, 100 + j)
    st.apply(b)
    F = f.apply_batch(b.u, b.v, b.new_cap, algo=algo); show(f"{algo} b{j} k={b.k}", F)
    f.min_cut_source_side(); print(f"    cut query {f.stats()['query_ms']:.3f} ms certified={f.stats()['certified']}", flush=True)
    check(st.graph(), F)
F = f.static_solve(); show("re-static", F)
F = f.static_solve_pp(); show("re-static-pp", F)
F = f.to_flow(); show("to_flow", F)
