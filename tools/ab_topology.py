"""A/B of the discharge schedule: worklist (async / rounds) vs topology-driven
vs the auto-switch, on static solves and 10% batches (config 4 bipartite, RMAT-20).
usage: python tools/ab_topology.py [bip|rmat20] [reps]"""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import workloads as W
import paper_2511_05895_b200 as P

which = sys.argv[1] if len(sys.argv) > 1 else "rmat20"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
if which == "bip":
    spec = dict(kind="bip", frac=0.10, nb=2, seed_base=400)
else:
    spec = dict(kind="rmat", scale=20, frac=0.10, nb=2, seed_base=100)
g, batches = W.sequence(spec)
sets = {"worklist(no switch)": dict(topo_div=-1), "auto(n/16)": dict(), "auto(n/64)": dict(topo_div=64),
        "topology": dict(schedule="topology"), "rounds(no switch)": dict(schedule="rounds", topo_div=-1)}
for rep in range(reps):
    for name, kn in sets.items():
        f = P.DynMaxFlow.from_graph(g, **kn)
        F = f.static_solve(); s0 = f.stats()
        row = {"static_ms": round(s0["device_ms"], 2), "topo_rounds": s0["topology_rounds"], "iters": s0["iterations"]}
        for j, b in enumerate(batches):
            for algo in ("pr", "pp"):
                pass
            f.apply_batch(b.u, b.v, b.new_cap, algo="pr" if j == 0 else "pp")
            s = f.stats()
            row[f"b{j}_{'pr' if j == 0 else 'pp'}_ms"] = round(s["device_ms"], 2)
            row[f"b{j}_topo"] = s["topology_rounds"]
        row["F"] = f.flow_value()
        print(f"{which} rep{rep} {name:22s} {json.dumps(row)}", flush=True)
        f.close()
