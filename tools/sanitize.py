"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck): config-1
graphs (CLRS chain + tiny random graphs, 10 mixed batches) and an RMAT-10 sequence under
every schedule, with F / S_min / S_max checked against brute force / Dinic.
usage: compute-sanitizer --tool memcheck python tools/sanitize.py [ngraphs]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import oracle as O
import workloads as W
import paper_2511_05895_b200 as P
from golden_io import graph, load

ng = int(sys.argv[1]) if len(sys.argv) > 1 else 12
fails = 0
def check(f, g, tag):
    global fails
    r = O.brute_force(g) if g.n <= 16 else O.maxflow(g, "dinic")
    ok = (f.flow_value() == r["F"] and np.array_equal(f.min_cut_source_side(), r["smin"])
          and np.array_equal(f.max_cut_source_side(), r["smax"]))
    if not ok:
        fails += 1
        print("MISMATCH", tag, flush=True)
for sched in ("async", "rounds", "topology"):
    g = graph(load("clrs_26_1.txt"))
    f = P.DynMaxFlow.from_graph(g, schedule=sched)
    f.static_solve(); check(f, g, f"{sched} clrs static")
    st = W.CapState(g)
    for j, step in enumerate(load("clrs_26_1.txt")["steps"]):
        b = W.as_batch(step["batch"]); st.apply(b)
        f.apply_batch(b.u, b.v, b.new_cap, algo="pp" if j % 2 else "pr"); check(f, st.graph(), f"{sched} clrs b{j}")
    f.to_flow()
    f.close()
    for seed in range(ng):
        g = W.tiny_random(seed)
        f = P.DynMaxFlow.from_graph(g, schedule=sched)
        f.static_solve(); check(f, g, f"{sched} tiny{seed}")
        st = W.CapState(g)
        for j, b in enumerate(W.tiny_batches(g, seed, nb=5)):
            st.apply(b)
            f.apply_batch(b.u, b.v, b.new_cap, algo="pp" if (seed + j) % 2 else "pr")
            check(f, st.graph(), f"{sched} tiny{seed} b{j}")
        f.close()
    g = W.rmat(10, 8, 1, 7)
    f = P.DynMaxFlow.from_graph(g, schedule=sched)
    f.static_solve(); check(f, g, f"{sched} rmat10")
    st = W.CapState(g)
    for j in range(3):
        b = W.rmat_batch(g, st, 0.02, 50 + j); st.apply(b)
        f.apply_batch(b.u, b.v, b.new_cap, algo="pp"); check(f, st.graph(), f"{sched} rmat10 b{j}")
    f.close()
# warm DYN_PP chains (F and S_min only: an S_max query would end the warm start), so the
# k_reach certificate, its failure path (MODE_PP_CONT), the back-off and the S_min query
# kernel all run under the tool
for knobs in (dict(), dict(schedule="async", budget_mul=-1000000, tail_items=1)):
    g = W.rmat(10, 8, 1, 7)
    f = P.DynMaxFlow.from_graph(g, **knobs)
    f.static_solve()
    st = W.CapState(g)
    seen = set()
    for j in range(8):
        b = W.rmat_batch(g, st, 0.01 if j % 2 else 0.002, 80 + j); st.apply(b)
        f.apply_batch(b.u, b.v, b.new_cap, algo="pp")
        seen.add(f.stats()["certified"])
        r = O.maxflow(st.graph(), "dinic")
        if not (f.flow_value() == r["F"] and np.array_equal(f.min_cut_source_side(), r["smin"])):
            fails += 1
            print("MISMATCH warm", knobs, j, flush=True)
    print("warm chain", knobs, "certificate outcomes", sorted(seen), flush=True)
    f.close()
print("sanitize workload done, mismatches:", fails)
