"""Debug: CLRS static solve under the async discharge; dump the debug event log."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import workloads as W
import paper_2511_05895_b200 as P
g = W.clrs_26_1()
for rep in range(3):
    f = P.DynMaxFlow.from_graph(g)
    f.set_trace(4096)
    F = f.static_solve()
    st = f.export_state()
    print("F", F, "res", st["res"].tolist(), "e", st["e"].tolist())
    cnt = ctypes.c_int32()
    f._check(f._L.dmf_get_trace(f._h, None, 0, ctypes.byref(cnt)))
    buf = np.zeros(8 * max(cnt.value, 1), np.int32)
    f._check(f._L.dmf_get_trace(f._h, P._ptr(buf), cnt.value, ctypes.byref(cnt)))
    names = {200: "START", 201: "END  ", 202: "ENQ  ", 203: "CLAIM"}
    rows = [r for r in buf[:8 * cnt.value].reshape(-1, 8) if r[0] >= 200]
    rows.sort(key=lambda r: int(r[6]))
    for r in rows:
        print(f"  {names[int(r[0])]} v={r[1]} warp={r[2]} a={r[3]} b={r[4]} c={r[5]} t={r[6]}")
    f.close()
    if F != 23: break
