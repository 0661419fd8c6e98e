"""Test-only helper: a plain numpy Bi-CSR slot layout (rows sorted by head, every
pair materialised, reverse index) used to hand the oracle's checker small states
written out by hand.  Independent of the CUDA library's builder."""
import numpy as np


def slots(n, edges):
    cap = {}
    for (u, v, c) in edges:
        cap[(u, v)] = cap.get((u, v), 0) + c
        cap.setdefault((v, u), 0)
    keys = sorted(cap)
    idx = {k: i for i, k in enumerate(keys)}
    row_ptr = np.zeros(n + 1, np.int64)
    for (u, _v) in keys:
        row_ptr[u + 1] += 1
    row_ptr = np.cumsum(row_ptr)
    dst = np.array([v for (_u, v) in keys], np.int32)
    rev = np.array([idx[(v, u)] for (u, v) in keys], np.int32)
    c = np.array([cap[k] for k in keys], np.int32)
    return row_ptr, dst, rev, c, idx


def state_from_flow(n, edges, netflow):
    """netflow: dict (u,v) -> net flow on the pair in direction u->v."""
    row_ptr, dst, rev, cap, idx = slots(n, edges)
    res = cap.astype(np.int64).copy()
    for (u, v), f in netflow.items():
        res[idx[(u, v)]] -= f
        res[idx[(v, u)]] += f
    e = np.zeros(n, np.int64)
    own = np.repeat(np.arange(n), np.diff(row_ptr))
    for i in range(len(dst)):
        e[dst[i]] += cap[i] - res[i]
    return row_ptr, dst, rev, cap, res.astype(np.int32), e
