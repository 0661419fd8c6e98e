import sys, os
sys.path.insert(0, "/root/repo")
sys.path.insert(0, "/root/repo/tests")
import numpy as np
import workloads as W
import oracle as O
from golden_io import graph, load
import paper_2511_05895_b200 as P
d = load("clrs_26_1.txt"); g = graph(d)
for name, kn in {"default": {}, "notopo": dict(topo_div=-1), "nogap": dict(local_gap=-1), "rounds": dict(schedule="rounds", topo_div=-1), "topo": dict(schedule="topology")}.items():
    for algo in ("pp", "pr"):
        f = P.DynMaxFlow.from_graph(g, **kn)
        f.static_solve()
        res = []
        for j, step in enumerate(d["steps"]):
            bb = W.as_batch(step["batch"])
            F = f.apply_batch(bb.u, bb.v, bb.new_cap, algo=algo)
            res.append((F, step["F"], f.to_flow()))
        print(name, algo, res, flush=True)
        f.close()
