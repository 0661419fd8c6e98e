"""Parser for tests/golden/*.txt fixtures (paper / textbook worked examples)."""
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    """Returns dict(n, s, t, edges[list of (u,v,c)], F, smin, smax, steps) where steps
    is a list of dict(fresh, batch, F, smin, smax) in file order."""
    d = dict(edges=[], steps=[])
    cur = None
    fresh = False
    for line in open(os.path.join(GOLDEN, name)):
        line = line.split("#", 1)[0].strip()
        if not line:
            continue
        key, _, rest = line.partition(" ")
        if key in ("n", "s", "t"):
            d[key] = int(rest)
        elif key == "edge":
            d["edges"].append(tuple(int(x) for x in rest.split()))
        elif key == "fresh":
            fresh = True
        elif key == "batch":
            ent = [tuple(int(x) for x in part.split()) for part in rest.split(";")]
            cur = dict(fresh=fresh, batch=ent)
            fresh = False
            d["steps"].append(cur)
        elif key in ("F", "smin", "smax"):
            tgt = d if cur is None else cur
            if key == "F":
                tgt["F"] = int(rest)
            else:
                m = np.zeros(d["n"], np.uint8)
                m[[int(x) for x in rest.split()]] = 1
                tgt[key] = m
    return d


def graph(d):
    import workloads as W
    a = np.array(d["edges"], np.int32)
    return W.Graph(d["n"], d["s"], d["t"], a[:, 0].copy(), a[:, 1].copy(), a[:, 2].copy(), name="golden")
