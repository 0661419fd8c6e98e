"""Debug build only (DMF_EXTRA_NVCC=-DDMF_DEBUG_BUSY DMF_LIB=.../libdmf_debug.so): event log
of the asynchronous discharge phase of warm DYN_PP batches on RMAT-`scale` ->
items in flight over time, per-item durations, ring waits (enqueue -> claim -> start)."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import workloads as W
import paper_2511_05895_b200 as P
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 6
g = W.rmat(scale, 16, 1, 7)
f = P.DynMaxFlow.from_graph(g)
f.static_solve()
cs = W.CapState(g)
deg = np.diff(np.concatenate([[0], np.cumsum(np.bincount(np.concatenate([g.u, g.v]), minlength=g.n))]))
for j in range(nb):
    b = W.rmat_batch(g, cs, 0.01, 100 + j); cs.apply(b)
    if j == nb - 1:
        f.set_trace(1 << 20)
    f.apply_batch(b.u, b.v, b.new_cap, algo="pp")
st = f.stats()
print("device ms", st["device_ms"], "discharge us", st["t_discharge_us"], "gap", st["gap_levels"], st["gap_skips"],
      "tail_stops", st["tail_stops"], "budget_stops", st["budget_stops"])
cnt = ctypes.c_int32()
f._check(f._L.dmf_get_trace(f._h, None, 0, ctypes.byref(cnt)))
buf = np.zeros(8 * max(cnt.value, 1), np.int32)
f._check(f._L.dmf_get_trace(f._h, P._ptr(buf), cnt.value, ctypes.byref(cnt)))
R = buf[:8 * cnt.value].reshape(-1, 8)
R = R[R[:, 0] >= 200]
t = R[:, 6].astype(np.int64)
t0 = t.min()
ts = (t - t0) / 1000.0
print("records", len(R), "span us", ts.max())
# items: start (200 vertex / 204 chunk) .. end (201 / 205) per warp
items = []
for w in np.unique(R[:, 2]):
    m = R[:, 2] == w
    rw, tw = R[m], ts[m]
    o = np.argsort(tw, kind="stable"); rw, tw = rw[o], tw[o]
    st_ = None
    for r, tt in zip(rw, tw):
        if r[0] in (200, 204): st_ = (tt, r)
        elif r[0] in (201, 205) and st_ is not None:
            items.append((st_[0], tt, int(st_[1][1]), int(st_[1][0]), int(r[5]) if r[0] == 201 else int(r[4])))
            st_ = None
items = np.array(items, dtype=np.float64)
print("items", len(items))
dur = items[:, 1] - items[:, 0]
for k, name in ((200, "vertex"), (204, "chunk")):
    sel = items[:, 3] == k
    d = dur[sel]
    if len(d):
        dg = deg[items[sel, 2].astype(int)]
        print(f"{name}: n={len(d)} dur p10={np.percentile(d,10):.1f} p50={np.median(d):.1f} p90={np.percentile(d, 90):.1f} max={d.max():.1f} us"
              f"  deg p50={np.median(dg):.0f} p90={np.percentile(dg,90):.0f}")
        for lo, hi in ((0, 2), (2, 8), (8, 17), (17, 128), (128, 513), (513, 1 << 30)):
            ss = (dg >= lo) & (dg < hi)
            if ss.sum():
                print(f"   deg [{lo},{hi}): n={ss.sum()} dur p50={np.median(d[ss]):.1f} p90={np.percentile(d[ss],90):.1f}")
# ring waits: enqueue (202, vertex a) -> claim (203, vertex a) -> next start of that vertex
enq = R[R[:, 0] == 202]; cl = R[R[:, 0] == 203]
te = {}
for r, tt in zip(enq, ts[R[:, 0] == 202]):
    te.setdefault(int(r[1]), []).append(tt)
waits = []
for r, tt in zip(cl, ts[R[:, 0] == 203]):
    lst = te.get(int(r[1]))
    if lst:
        prev = [x for x in lst if x <= tt]
        if prev: waits.append(tt - prev[-1])
if waits:
    w = np.array(waits)
    print(f"enqueue->claim wait: n={len(w)} p50={np.median(w):.2f} p90={np.percentile(w,90):.2f} max={w.max():.1f} us")
lab = f.export_labels()
vs, cnts = np.unique(items[:, 2].astype(np.int64), return_counts=True)
o = np.argsort(-cnts)[:15]
print("top vertices by items: (v, items, deg, part, e-sign, hp, hm)")
ex = f.export_state()["e"]
for i in o:
    v = vs[i]
    print(f"   v={v} items={cnts[i]} deg={deg[v]} part={lab['part'][v]} e={ex[v]} hp={lab['hp'][v]} hm={lab['hm'][v]} s={v == g.s} t={v == g.t}")
print("distinct vertices", len(vs), "chunk vertices", len(np.unique(items[items[:, 3] == 204, 2])))
edges = np.arange(0, ts.max() + 10, 10)
for lo in edges:
    hi = lo + 10
    fl = ((items[:, 0] < hi) & (items[:, 1] > lo)).sum()
    stt = ((items[:, 0] >= lo) & (items[:, 0] < hi)).sum()
    print(f"  t={lo:6.0f}-{hi:<6.0f} in-flight {fl:5d} started {stt:5d}")

# ---- critical path: each item's predecessor = the item whose warp enqueued its vertex
# (the latest enqueue of that vertex before the item's claim)
enq_rows = R[R[:, 0] == 202]
enq_t = ts[R[:, 0] == 202]
claim_rows = R[R[:, 0] == 203]
claim_t = ts[R[:, 0] == 203]
# item intervals per warp, to map (warp, time) -> item index
order = np.lexsort((items[:, 0], ))
by_warp = {}
item_warp = []
for idx, (a, b, v, k, x) in enumerate(items):
    pass
# rebuild items with warp ids
items2 = []
for w in np.unique(R[:, 2]):
    m = R[:, 2] == w
    rw, tw = R[m], ts[m]
    o = np.argsort(tw, kind="stable"); rw, tw = rw[o], tw[o]
    st_ = None
    for r, tt in zip(rw, tw):
        if r[0] in (200, 204): st_ = (tt, r)
        elif r[0] in (201, 205) and st_ is not None:
            items2.append((st_[0], tt, int(st_[1][1]), int(st_[1][0]), int(w)))
            st_ = None
items2.sort()
I = np.array(items2, dtype=np.float64)
from collections import defaultdict
warp_items = defaultdict(list)
for idx, it in enumerate(items2):
    warp_items[it[4]].append((it[0], it[1], idx))
def item_at(w, t):
    for a, b, idx in warp_items.get(w, []):
        if a - 0.01 <= t <= b + 0.01:
            return idx
    return -1
# enqueues of vertex v: (time, producing item)
enq_by_v = defaultdict(list)
for r, tt in zip(enq_rows, enq_t):
    enq_by_v[int(r[1])].append((tt, item_at(int(r[2]), tt)))
pred = np.full(len(items2), -1)
for idx, (a, b, v, kind, w) in enumerate(items2):
    lst = [x for x in enq_by_v.get(v, []) if x[0] <= a]
    if lst:
        pred[idx] = lst[-1][1]
# longest chain ending at each item by end time
dist = np.zeros(len(items2))
for idx in range(len(items2)):
    p = pred[idx]
    dist[idx] = (items2[idx][1] - items2[idx][0]) + (dist[p] if p >= 0 else 0)
# the stage-1 phase: items before the first idle gap of >= 20 us
srt = np.argsort(I[:, 0])
cut_t = I[:, 1].max()
run_end = I[srt[0], 1]
for ii in srt:
    if I[ii, 0] > run_end + 20:
        cut_t = run_end; break
    run_end = max(run_end, I[ii, 1])
sel = np.nonzero(I[:, 1] <= cut_t + 0.01)[0]
end = int(sel[np.argmax(I[sel, 1])])
print(f"phase ends at {I[end, 1]:.1f} us ({len(sel)} items); last item's chain busy time {dist[end]:.1f} us; "
      f"max chain busy {dist[sel].max():.1f} us")
chain = []
c = end
while c >= 0 and len(chain) < 200:
    chain.append(c); c = pred[c]
chain = chain[::-1]
print(f"critical chain: {len(chain)} items")
for c in chain[-60:]:
    a, b, v, kind, w = items2[c]
    print(f"   t={a:7.1f}-{b:7.1f} ({b-a:5.1f} us) {'chunk' if kind == 204 else 'vertex'} v={v} deg={deg[v]} part={lab['part'][v]} hp={lab['hp'][v]} hm={lab['hm'][v]}")
