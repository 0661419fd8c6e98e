"""A/B of engine knobs on the bench sequence (RMAT-`scale`, static solve, cumulative 1%
mixed PP batches): median device ms per batch and per phase, per knob set.
usage: python tools/ab.py SCALE NBATCH 'name:k=v,k=v' 'name2:...' ..."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import workloads as W
import paper_2511_05895_b200 as P

scale = int(sys.argv[1]); nb = int(sys.argv[2])
sets = []
for a in sys.argv[3:]:
    name, _, kv = a.partition(":")
    kn = {}
    for item in filter(None, kv.split(",")):
        k, v = item.split("=")
        kn[k] = v if k == "schedule" else int(v)
    sets.append((name, kn))
g = W.rmat(scale, 16, 1, 7)
cs = W.CapState(g)
batches = []
for j in range(nb):
    b = W.rmat_batch(g, cs, 0.01, 100 + j); cs.apply(b); batches.append(b)
keys = ("t_prologue_us", "t_reset_us", "t_bfs_us", "t_discharge_us", "t_rie_us", "t_epilogue_us")
for rep in range(2):
    for name, kn in sets:
        f = P.DynMaxFlow.from_graph(g, **kn)
        f.static_solve(); st0 = f.stats()
        f.static_solve_pp(); st1 = f.stats()
        per = []; cut = []
        import torch
        mask = torch.empty(g.n, dtype=torch.uint8, device="cuda")
        for j, b in enumerate(batches):
            f.apply_batch(b.u, b.v, b.new_cap, algo="pp")
            if j >= 5:
                per.append(f.stats())
            if not os.environ.get("AB_NO_CUT"):
                t0 = time.perf_counter()
                f.min_cut_source_side(mask)
                if j >= 5:
                    cut.append(1e3 * (time.perf_counter() - t0))
        ms = [p["device_ms"] for p in per]
        med = {k: round(float(np.median([p[k] for p in per])), 1) for k in keys}
        ex = {k: float(np.mean([p[k] for p in per])) for k in ("iterations", "gap_levels", "gap_skips", "tail_stops",
                                                                 "budget_stops", "stage2_skipped", "discharge_vertices", "certified")}
        print(f"{name:14s} rep{rep} cut ms p50={np.median(cut) if cut else 0:.3f} batch ms p50={np.median(ms):.3f} p90={np.percentile(ms, 90):.3f} mean={np.mean(ms):.3f} "
              f"static alg1={st0['device_ms']:.2f} pp={st1['device_ms']:.2f}  {med}  {json.dumps({k: round(v, 2) for k, v in ex.items()})}",
              flush=True)
        f.close()
