"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2511_05895_b200``) never imports it, and it never imports the product.

Contents (each function cites the passage it follows; see oracle/oracle.c):

* ``maxflow(g, algo)`` -- F, S_min, S_max, per-edge flow by Edmonds-Karp, Dinitz or
  two-phase FIFO push-relabel (definition of max-flow / min-cut).
* ``brute_force(g)`` -- enumerates every s-t cut of a graph with n <= 16 (numpy):
  F = min cut capacity (max-flow min-cut theorem), S_min = intersection and
  S_max = union of all minimising source sides.
* ``hopcroft_karp(nl, nr, l, r)`` -- maximum bipartite matching (config 4 pin).
* ``grid_terminal_closed_form(cs, ct)`` -- terminal-only grid: F = sum min(c_s, c_t).
* ``check_state(...)`` -- certificate / invariant checker of an exported solver state
  (capacity, pair-sum, excess, no augmenting path, conversion to a true flow and its
  conservation, S_min and cut capacity; Thm 3, Lemma 4 P:276-304,
  Lemma P:411-443).

Parity pins: every function above is pinned in tests/test_oracle.py against
textbook worked examples (CLRS Fig. 26.1, SPEC G1), brute force, closed forms,
scipy's independent max-flow, Hopcroft-Karp and weak duality.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

EK, DINIC, FIFO_PR = 0, 1, 2
ALGOS = {"ek": EK, "dinic": DINIC, "fifo_pr": FIFO_PR}


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (plain C, -O2)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", _LIB, _SRC])
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        L.orc_maxflow.restype = ctypes.c_int64
        L.orc_maxflow.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int64, P, P, P,
                                  ctypes.c_int32, ctypes.c_int32, P, P, P, P]
        L.orc_hopcroft_karp.restype = ctypes.c_int64
        L.orc_hopcroft_karp.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int64, P, P]
        L.orc_check_state.restype = ctypes.c_int
        L.orc_check_state.argtypes = [ctypes.c_int32, ctypes.c_int64, P, P, P, P, P, P,
                                      ctypes.c_int32, ctypes.c_int32, ctypes.c_int64, P,
                                      ctypes.c_char_p, ctypes.c_int32, P]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def maxflow(g, algo: str = "dinic", want_flow: bool = False, stats: bool = False):
    """Max flow of graph ``g`` (workloads.Graph-like: n, s, t, u, v, cap).

    Returns dict(F, smin (uint8[n]), smax (uint8[n]), flow (int64[m] or None),
    stats).  S_min = reach from s in the final residual graph of a true maximum
    flow; S_max = V minus the vertices that reach t."""
    L = _load()
    u = np.ascontiguousarray(g.u, np.int32)
    v = np.ascontiguousarray(g.v, np.int32)
    c = np.ascontiguousarray(g.cap, np.int32)
    smin = np.zeros(g.n, np.uint8)
    smax = np.zeros(g.n, np.uint8)
    flow = np.zeros(len(u), np.int64) if want_flow else None
    st = np.zeros(4, np.int64)
    F = L.orc_maxflow(ALGOS[algo], g.n, len(u), _p(u), _p(v), _p(c), g.s, g.t,
                      _p(smin), _p(smax), _p(flow), _p(st))
    if F < 0:
        raise RuntimeError(f"oracle maxflow failed ({F})")
    return dict(F=int(F), smin=smin, smax=smax, flow=flow,
                stats=dict(pushes=int(st[0]), relabels=int(st[1]), gaps=int(st[2]), global_relabels=int(st[3])))


def hopcroft_karp(nl: int, nr: int, l: np.ndarray, r: np.ndarray) -> int:
    """Maximum matching size of the bipartite graph with edges (l[j], r[j])."""
    L = _load()
    l = np.ascontiguousarray(l, np.int32)
    r = np.ascontiguousarray(r, np.int32)
    return int(L.orc_hopcroft_karp(nl, nr, len(l), _p(l), _p(r)))


def check_state(n, s, t, row_ptr, dst, rev, cap, res, e, F, smin=None, want_flow=False):
    """Run the C checker on an exported slot-form state.  Returns (code, message,
    converted_residuals or None); code 0 = every check passed."""
    L = _load()
    row_ptr = np.ascontiguousarray(row_ptr, np.int64)
    dst = np.ascontiguousarray(dst, np.int32)
    rev = np.ascontiguousarray(rev, np.int32)
    cap = np.ascontiguousarray(cap, np.int32)
    res = np.ascontiguousarray(res, np.int32)
    e = np.ascontiguousarray(e, np.int64)
    sm = None if smin is None else np.ascontiguousarray(smin, np.uint8)
    buf = ctypes.create_string_buffer(512)
    out = np.zeros(len(dst), np.int32) if want_flow else None
    rc = L.orc_check_state(n, len(dst), _p(row_ptr), _p(dst), _p(rev), _p(cap), _p(res), _p(e),
                           s, t, int(F), _p(sm), buf, 512, _p(out))
    return int(rc), buf.value.decode(), out


def cap_matrix(g) -> np.ndarray:
    """Dense n x n capacity matrix (parallel edges summed, self-loops dropped)."""
    C = np.zeros((g.n, g.n), np.int64)
    keep = g.u != g.v
    np.add.at(C, (g.u[keep], g.v[keep]), g.cap[keep].astype(np.int64))
    return C


def brute_force(g):
    """Enumerate all 2^(n-2) s-t cuts (n <= 16).  cap(S) = sum_{u in S, v not in S}
    c(u,v).  By max-flow min-cut F = min cap(S); S_min / S_max are the
    intersection / union of the minimising source sides."""
    n, s, t = g.n, g.s, g.t
    assert n <= 16
    C = cap_matrix(g)
    others = [x for x in range(n) if x not in (s, t)]
    k = len(others)
    masks = np.arange(1 << k, dtype=np.int64)
    M = np.zeros((1 << k, n), np.int64)
    M[:, s] = 1
    for j, x in enumerate(others):
        M[:, x] = (masks >> j) & 1
    caps = ((M @ C) * (1 - M)).sum(axis=1)
    F = int(caps.min())
    best = M[caps == F].astype(bool)
    return dict(F=F, smin=best.all(axis=0).astype(np.uint8), smax=best.any(axis=0).astype(np.uint8))


def grid_terminal_closed_form(cs: np.ndarray, ct: np.ndarray):
    """Terminal-only grid (no n-links): each pixel p is an independent path
    s->p->t, so F = sum_p min(c(s,p), c(p,t)) and S_min = {s} u {p : c(s,p) > c(p,t)}
    (the s-p edge is not saturated iff c(s,p) > c(p,t))."""
    cs = cs.astype(np.int64)
    ct = ct.astype(np.int64)
    return int(np.minimum(cs, ct).sum()), (cs > ct)
