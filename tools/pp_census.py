"""Census of the converged state after each DYN_PP batch (bench sequence): sizes of the
partition, excess / deficit vertices by side, |S_min|, and the stats of the batch."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import workloads as W
import paper_2511_05895_b200 as P
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 8
g, batches = W.sequence(dict(kind="rmat", scale=scale, frac=0.01, nb=nb))
f = P.DynMaxFlow.from_graph(g)
f.static_solve()
n = g.n
for j, b in enumerate(batches):
    f.apply_batch(b.u, b.v, b.new_cap, algo="pp")
    st = f.stats()
    lab = f.export_labels(); e = f.export_state()["e"]
    part = lab["part"]; hp = lab["hp"]; hm = lab["hm"]
    smin = f.min_cut_source_side()
    T = part == 2; S = part == 1
    off = np.ones(n, bool); off[[g.s, g.t]] = False
    print(f"b{j}: ms={st['device_ms']:.3f} |T|={T.sum()} |S|={S.sum()} |Smin|={smin.sum()} "
          f"exc S={((e > 0) & S & off).sum()} T={((e > 0) & T & off).sum()} def S={((e < 0) & S & off).sum()} "
          f"T={((e < 0) & T & off).sum()} hm<n in S={((hm < n) & S).sum()} maxhp={hp[T].max() if T.any() else -1} "
          f"maxhm={hm[(hm < n)].max()} s2={st['stage2_vertices']} s2it={st['stage2_iterations']} it={st['iterations']} "
          f"gap={st['gap_levels']}/{st['gap_skips']}", flush=True)
