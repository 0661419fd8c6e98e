"""Debug build only (-DDMF_DEBUG_BUSY): event log of the asynchronous discharge phase of a
warm DYN_PP batch on RMAT-20 -> items in flight over time and per-item durations."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import workloads as W
import paper_2511_05895_b200 as P
g = W.rmat(20, 16, 1, 7)
f = P.DynMaxFlow.from_graph(g)
f.static_solve()
cs = W.CapState(g)
for j in range(3):
    b = W.rmat_batch(g, cs, 0.01, 100 + j); cs.apply(b)
    if j == 2:
        f.set_trace(1 << 17)
    f.apply_batch(b.u, b.v, b.new_cap, algo="pp")
print("device ms", f.stats()["device_ms"], "discharge us", f.stats()["t_discharge_us"])
cnt = ctypes.c_int32()
f._check(f._L.dmf_get_trace(f._h, None, 0, ctypes.byref(cnt)))
buf = np.zeros(8 * max(cnt.value, 1), np.int32)
f._check(f._L.dmf_get_trace(f._h, P._ptr(buf), cnt.value, ctypes.byref(cnt)))
R = buf[:8 * cnt.value].reshape(-1, 8)
R = R[R[:, 0] >= 200]
t = R[:, 6].astype(np.int64)
t0 = t.min()
ts = (t - t0) / 1000.0
kinds = R[:, 0]
# pair starts / ends per warp (records of one warp are sequential)
items = []
for w in np.unique(R[:, 2]):
    m = R[:, 2] == w
    rw, tw = R[m], ts[m]
    o = np.argsort(tw, kind="stable"); rw, tw = rw[o], tw[o]
    st = None
    for r, tt in zip(rw, tw):
        if r[0] in (200, 204): st = (tt, r)
        elif r[0] in (201, 205) and st is not None:
            items.append((st[0], tt, int(st[1][1]), int(st[1][0])))
            st = None
items = np.array([(a, b, v, k) for a, b, v, k in items])
print("items", len(items), "span us", ts.max())
dur = items[:, 1] - items[:, 0]
for k, name in ((200, "vertex"), (204, "chunk")):
    d = dur[items[:, 3] == k]
    if len(d): print(f"{name}: n={len(d)} dur p50={np.median(d):.1f} p90={np.percentile(d, 90):.1f} max={d.max():.1f} us")
edges = np.arange(0, ts.max() + 10, 10)
for lo in edges:
    hi = lo + 10
    fl = ((items[:, 0] < hi) & (items[:, 1] > lo)).sum()
    st = ((items[:, 0] >= lo) & (items[:, 0] < hi)).sum()
    print(f"  t={lo:6.0f}-{hi:<6.0f} in-flight {fl:5d} started {st:5d}")
