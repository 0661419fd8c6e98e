"""Seeded synthetic inputs shared by the CUDA path, the oracle, the tests and bench.py.

This module holds NO arithmetic of the method (no residuals, no excess, no heights,
no flows): it only draws graphs and capacity-update batches, deterministically from
integer seeds, with the shapes SURVEY.md §8(d) lists for the five BASELINE.json
configs.  Both sides (the CUDA library through ``paper_2511_05895_b200`` and the
CPU oracle under ``oracle/``) consume its outputs; neither side is imported here.

Conventions
-----------
* A graph is ``Graph(n, s, t, u, v, cap)``: directed input edges (int32 arrays),
  no self-loops, no duplicate ordered pairs, capacities >= 0 (zero-capacity input
  edges are kept: they are the insert pool, "a jump from zero capacity to a
  positive capacity simulates addition of an edge").
* A batch is ``Batch(u, v, new_cap)`` (int32 arrays): SET semantics, all entries
  simultaneous, no duplicate (u, v).
* ``CapState`` tracks the cumulative capacity of every ordered pair so that a batch
  generator can draw "higher or lower" values and so that the oracle can be
  handed the current edge list for a full recompute after every batch.

Randomness: numpy ``Generator(PCG64(seed))`` -- deterministic across platforms.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

__all__ = [
    "Graph", "Batch", "CapState",
    "clrs_26_1", "spec_g1", "tiny_random", "tiny_batches",
    "rmat", "rmat_batch", "grid", "grid_batch", "bipartite", "bipartite_batch",
    "to_csr", "config_graph",
]


@dataclasses.dataclass
class Graph:
    n: int
    s: int
    t: int
    u: np.ndarray      # int32[m]
    v: np.ndarray      # int32[m]
    cap: np.ndarray    # int32[m]
    name: str = ""
    meta: dict = dataclasses.field(default_factory=dict)

    @property
    def m(self) -> int:
        return int(self.u.shape[0])


@dataclasses.dataclass
class Batch:
    u: np.ndarray      # int32[k]
    v: np.ndarray      # int32[k]
    new_cap: np.ndarray  # int32[k]

    @property
    def k(self) -> int:
        return int(self.u.shape[0])


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(int(seed)))


def _unique_sorted(key: np.ndarray) -> np.ndarray:
    """Sorted distinct values (np.unique is hash-based and slow on 10^7+ int64)."""
    key = np.sort(key)
    if key.shape[0] == 0:
        return key
    keep = np.empty(key.shape[0], bool)
    keep[0] = True
    np.not_equal(key[1:], key[:-1], out=keep[1:])
    return key[keep]


def to_csr(g: Graph):
    """CSR (row_ptr int64[n+1], col int32[m], cap int32[m]) of the input edge list,
    rows in vertex order, edges of a row in input order (stable sort by tail)."""
    order = np.argsort(g.u, kind="stable")
    counts = np.bincount(g.u, minlength=g.n).astype(np.int64)
    row_ptr = np.zeros(g.n + 1, np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    return row_ptr, np.ascontiguousarray(g.v[order], np.int32), np.ascontiguousarray(g.cap[order], np.int32)


class CapState:
    """Current capacity of every ordered pair (u, v) that is an input edge or the
    reverse of one.  Pure bookkeeping of SET-semantics updates (no method maths)."""

    def __init__(self, g: Graph):
        self.n = g.n
        self.s, self.t = g.s, g.t
        key = g.u.astype(np.int64) * g.n + g.v.astype(np.int64)
        order = np.argsort(key, kind="stable")
        self.key = key[order]
        self.cap = g.cap[order].astype(np.int64)
        self.extra: dict[int, int] = {}   # reverse pairs touched by a batch

    def lookup(self, u: np.ndarray, v: np.ndarray) -> np.ndarray:
        k = u.astype(np.int64) * self.n + v.astype(np.int64)
        pos = np.searchsorted(self.key, k)
        pos_c = np.minimum(pos, len(self.key) - 1)
        hit = (pos < len(self.key)) & (self.key[pos_c] == k)
        out = np.where(hit, self.cap[pos_c], 0)
        if self.extra:
            for i in np.nonzero(~hit)[0]:
                out[i] = self.extra.get(int(k[i]), 0)
        return out

    def apply(self, b: Batch) -> None:
        k = b.u.astype(np.int64) * self.n + b.v.astype(np.int64)
        pos = np.searchsorted(self.key, k)
        pos_c = np.minimum(pos, len(self.key) - 1)
        hit = (pos < len(self.key)) & (self.key[pos_c] == k)
        self.cap[pos_c[hit]] = b.new_cap[hit]
        for i in np.nonzero(~hit)[0]:
            self.extra[int(k[i])] = int(b.new_cap[i])

    def edges(self):
        """(u, v, cap) int32 arrays of the current capacities, including touched
        reverse pairs (zero-capacity pairs are kept)."""
        keys = self.key
        caps = self.cap
        if self.extra:
            ek = np.fromiter(self.extra.keys(), np.int64, len(self.extra))
            ec = np.fromiter(self.extra.values(), np.int64, len(self.extra))
            keys = np.concatenate([keys, ek])
            caps = np.concatenate([caps, ec])
        u = (keys // self.n).astype(np.int32)
        v = (keys % self.n).astype(np.int32)
        return u, v, caps.astype(np.int32)

    def graph(self) -> Graph:
        u, v, c = self.edges()
        return Graph(self.n, self.s, self.t, u, v, c, name="capstate")


# ----------------------------------------------------------------------------
# config 1: textbook + tiny random graphs
# ----------------------------------------------------------------------------

def clrs_26_1() -> Graph:
    """CLRS 3e Fig. 26.1 flow network. Vertex ids: s=0, v1=1, v2=2, v3=3, v4=4, t=5."""
    e = [(0, 1, 16), (0, 2, 13), (1, 3, 12), (2, 1, 4), (2, 4, 14),
         (3, 2, 9), (3, 5, 20), (4, 3, 7), (4, 5, 4)]
    a = np.array(e, np.int32)
    return Graph(6, 0, 5, a[:, 0].copy(), a[:, 1].copy(), a[:, 2].copy(), name="clrs_26_1")


CLRS_CHAIN = [  # cumulative batches on CLRS Fig. 26.1 (ids as in clrs_26_1)
    [(4, 5, 10)],
    [(1, 3, 5)],
    [(0, 1, 0), (3, 5, 25)],
    [(4, 3, 0), (2, 4, 20), (5, 3, 7)],
    [(3, 1, 6)],
]


def spec_g1() -> Graph:
    """SPEC.md S:64 example G1 = {(0,1,4),(0,2,2),(1,2,3),(1,3,1),(2,3,6)}, s=0, t=3."""
    a = np.array([(0, 1, 4), (0, 2, 2), (1, 2, 3), (1, 3, 1), (2, 3, 6)], np.int32)
    return Graph(4, 0, 3, a[:, 0].copy(), a[:, 1].copy(), a[:, 2].copy(), name="spec_g1")


def as_batch(entries) -> Batch:
    a = np.array(entries, np.int32).reshape(-1, 3)
    return Batch(a[:, 0].copy(), a[:, 1].copy(), a[:, 2].copy())


def tiny_random(seed: int, nmin: int = 2, nmax: int = 12, p: float = 0.35, capmax: int = 10) -> Graph:
    """Config 1 random graph: n ~ U{nmin..nmax}, every ordered pair
    present with probability p, cap ~ U{1..capmax}, s=0, t=n-1."""
    r = _rng(seed)
    n = int(r.integers(nmin, nmax + 1))
    uu, vv = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    mask = (uu != vv) & (r.random((n, n)) < p)
    u = uu[mask].astype(np.int32)
    v = vv[mask].astype(np.int32)
    cap = r.integers(1, capmax + 1, size=u.shape[0]).astype(np.int32)
    return Graph(n, 0, n - 1, u, v, cap, name=f"tiny{seed}")


def _pair_slots(g: Graph):
    """All materialised ordered pairs: input edges and their reverses (sorted keys)."""
    k1 = g.u.astype(np.int64) * g.n + g.v
    k2 = g.v.astype(np.int64) * g.n + g.u
    return _unique_sorted(np.concatenate([k1, k2]))


def tiny_batches(g: Graph, seed: int, nb: int = 10, incmax: int = 10):
    """Config 1 batches: nb cumulative mixed batches; k ~ U{1..max(1,S//3)} distinct
    slots drawn from ALL materialised pairs (so 0 -> c insertions happen); the first
    ceil(k/2) are increments U[old+1, old+incmax], the rest decrements U[0, old-1]
    (a decrement of a zero-capacity pair stays 0).  Yields Batch objects; the caller
    applies them to its CapState (the generator keeps its own copy)."""
    r = _rng(10_000 + seed)
    slots = _pair_slots(g)
    st = CapState(g)
    out = []
    if len(slots) == 0:
        return [Batch(np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros(0, np.int32)) for _ in range(nb)]
    for _ in range(nb):
        S = len(slots)
        k = int(r.integers(1, max(1, S // 3) + 1))
        pick = r.choice(S, size=k, replace=False)
        keys = slots[pick]
        u = (keys // g.n).astype(np.int32)
        v = (keys % g.n).astype(np.int32)
        old = st.lookup(u, v)
        ninc = (k + 1) // 2
        new = np.empty(k, np.int64)
        new[:ninc] = old[:ninc] + r.integers(1, incmax + 1, size=ninc)
        dec_old = old[ninc:]
        new[ninc:] = np.where(dec_old > 0, np.floor(r.random(k - ninc) * np.maximum(dec_old, 1)).astype(np.int64), 0)
        b = Batch(u, v, new.astype(np.int32))
        st.apply(b)
        out.append(b)
    return out


# ----------------------------------------------------------------------------
# config 2 / 5: RMAT power-law graphs
# ----------------------------------------------------------------------------

def rmat(scale: int = 20, edge_factor: int = 16, seed_graph: int = 1, seed_caps: int = 7,
         capmax: int = 1000, abc=(0.57, 0.19, 0.19)) -> Graph:
    """Graph500-style RMAT: 2^scale vertices, edge_factor*2^scale
    draws with quadrant probabilities (a,b,c,d), random vertex permutation, self-loops
    dropped, duplicate pairs removed; caps U[1,capmax]; s = argmax out-degree,
    t = argmax in-degree (!= s)."""
    n = 1 << scale
    M = edge_factor << scale
    r = _rng(seed_graph)
    a, b, c = abc
    u = np.zeros(M, np.int64)
    v = np.zeros(M, np.int64)
    for bit in range(scale):
        x = r.random(M, dtype=np.float32)
        ub = x >= (a + b)
        vb = ((x >= a) & (x < a + b)) | (x >= a + b + c)
        u |= ub.astype(np.int64) << bit
        v |= vb.astype(np.int64) << bit
        del x, ub, vb
    perm = r.permutation(n).astype(np.int64)
    u = perm[u]
    v = perm[v]
    keep = u != v
    key = _unique_sorted(u[keep] * n + v[keep])
    del u, v, keep
    u = (key // n).astype(np.int32)
    v = (key % n).astype(np.int32)
    cap = _rng(seed_caps).integers(1, capmax + 1, size=key.shape[0]).astype(np.int32)
    outdeg = np.bincount(u, minlength=n)
    indeg = np.bincount(v, minlength=n)
    s = int(np.argmax(outdeg))
    indeg_t = indeg.copy()
    indeg_t[s] = -1
    t = int(np.argmax(indeg_t))
    return Graph(n, s, t, u, v, cap, name=f"rmat{scale}",
                 meta=dict(scale=scale, edge_factor=edge_factor, seed_graph=seed_graph, seed_caps=seed_caps))


def _weighted_sample(r: np.random.Generator, w: np.ndarray, k: int) -> np.ndarray:
    """k distinct indices, weighted sampling without replacement (Efraimidis-Spirakis
    keys log(U)/w, top-k), returned in a random order."""
    m = w.shape[0]
    k = min(k, m)
    keys = np.log(r.random(m)) / w
    idx = np.argpartition(-keys, k - 1)[:k] if k < m else np.arange(m)
    idx = np.sort(idx)
    return idx[r.permutation(k)]


def _weighted_sample_two_class(r: np.random.Generator, m: int, heavy: np.ndarray, bias: float, k: int) -> np.ndarray:
    """The same distribution as _weighted_sample (Efraimidis-Spirakis top-k of
    log(U)/w) when every weight is 1 except weight `bias` on the sorted indices
    `heavy`, in O(k + |heavy|) instead of O(m): the heavy keys are drawn as they are;
    of the weight-1 class only its k largest keys can reach the overall top k, and the
    k largest of M iid log(U) are -(Z_1/M + Z_2/(M-1) + ...) (Exp(1) spacings, Renyi)
    sitting on a uniformly random k-subset of the class (ranks independent of values)."""
    k = min(k, m)
    nh = heavy.shape[0]
    ma = m - nh
    kh = np.log(r.random(nh)) / bias
    ka_n = min(k, ma)
    z = r.exponential(1.0, size=ka_n) / (ma - np.arange(ka_n, dtype=np.float64))
    ka = -np.cumsum(z)
    pos = r.choice(ma, size=ka_n, replace=False) if ka_n else np.zeros(0, np.int64)
    # pos-th element of the light class = pos + number of heavy indices before it
    shift = heavy - np.arange(nh)
    a_idx = pos + np.searchsorted(shift, pos, side="right")
    keys = np.concatenate([kh, ka])
    cand = np.concatenate([heavy.astype(np.int64), a_idx.astype(np.int64)])
    top = np.argpartition(-keys, k - 1)[:k] if k < keys.shape[0] else np.arange(keys.shape[0])
    idx = np.sort(cand[top])
    return idx[r.permutation(idx.shape[0])]


def rmat_batch(g: Graph, st: CapState, frac: float, seed: int, kind: str = "mix",
               bias: float = 10.0, capmax: int = 1000) -> Batch:
    """Batch of round(frac*m) distinct existing input edges, weight `bias` on
    edges leaving s or entering t; inc U[old+1, old+capmax], dec U[0, old-1]
    (R20); mix = ceil(k/2) inc + floor(k/2) dec."""
    r = _rng(seed)
    k = max(1, int(round(frac * g.m)))
    heavy = g.meta.get("_heavy")
    if heavy is None:
        heavy = np.nonzero((g.u == g.s) | (g.v == g.t))[0]
        g.meta["_heavy"] = heavy
    idx = _weighted_sample_two_class(r, g.m, heavy, bias, k)
    u = g.u[idx]
    v = g.v[idx]
    old = st.lookup(u, v)
    k = idx.shape[0]
    ninc = {"mix": (k + 1) // 2, "inc": k, "dec": 0}[kind]
    new = np.empty(k, np.int64)
    new[:ninc] = old[:ninc] + r.integers(1, capmax + 1, size=ninc)
    dold = old[ninc:]
    new[ninc:] = np.where(dold > 0, np.floor(r.random(k - ninc) * np.maximum(dold, 1)).astype(np.int64), 0)
    return Batch(u.astype(np.int32), v.astype(np.int32), new.astype(np.int32))


# ----------------------------------------------------------------------------
# config 3: image-segmentation grid
# ----------------------------------------------------------------------------

def _grid_image(W: int, r: np.random.Generator) -> np.ndarray:
    yy, xx = np.mgrid[0:W, 0:W]
    img = np.full((W, W), 60.0)
    for _ in range(8):
        rad = r.uniform(W / 16, W / 4)
        cy, cx = r.uniform(0, W, size=2)
        img[(yy - cy) ** 2 + (xx - cx) ** 2 <= rad * rad] = 190.0
    img += r.normal(0.0, 40.0, size=(W, W))
    return np.clip(img, 0, 255)


def _tlinks(I: np.ndarray):
    cs = np.rint(1000.0 * I / 255.0).astype(np.int32)
    ct = np.rint(1000.0 * (255.0 - I) / 255.0).astype(np.int32)
    return cs, ct


def grid(W: int = 2048, seed: int = 3, nlinks: bool = True) -> Graph:
    """Config 3: W*W pixels (ids y*W+x), s = W*W, t = W*W+1.
    t-links c(s,p)=round(1000 I/255), c(p,t)=round(1000(255-I)/255); 4-neighbour
    n-links in both directions with cap 1+round(100 exp(-dI^2/(2*30^2)))."""
    r = _rng(seed)
    I = _grid_image(W, r)
    npx = W * W
    s, t = npx, npx + 1
    cs, ct = _tlinks(I.ravel())
    pid = np.arange(npx, dtype=np.int64).reshape(W, W)
    us = [np.full(npx, s, np.int64), pid.ravel()]
    vs = [pid.ravel(), np.full(npx, t, np.int64)]
    cps = [cs, ct]
    if nlinks:
        for (dy, dx) in ((0, 1), (1, 0)):
            a = pid[: W - dy, : W - dx].ravel()
            b = pid[dy:, dx:].ravel()
            Ia = I[: W - dy, : W - dx].ravel()
            Ib = I[dy:, dx:].ravel()
            c = (1 + np.rint(100.0 * np.exp(-((Ia - Ib) ** 2) / (2 * 30.0 ** 2)))).astype(np.int32)
            us += [a, b]
            vs += [b, a]
            cps += [c, c]
    u = np.concatenate(us).astype(np.int32)
    v = np.concatenate(vs).astype(np.int32)
    cap = np.concatenate(cps).astype(np.int32)
    return Graph(npx + 2, s, t, u, v, cap, name=f"grid{W}",
                 meta=dict(W=W, seed=seed, image=I.astype(np.float32)))


def grid_batch(g: Graph, frac: float, seed: int) -> Batch:
    """Perturb round(frac*W*W) distinct pixels I' = clip(I + N(0,60)) and set both
    t-links from I' (2 entries per pixel, mixed inc/dec).  Intensities drift
    cumulatively: g.meta['image'] is updated in place."""
    r = _rng(seed)
    W = g.meta["W"]
    I = g.meta["image"].ravel()
    npx = W * W
    k = max(1, int(round(frac * npx)))
    px = np.sort(r.choice(npx, size=k, replace=False))
    Ip = np.clip(I[px] + r.normal(0.0, 60.0, size=k), 0, 255)
    I[px] = Ip
    cs, ct = _tlinks(Ip)
    u = np.concatenate([np.full(k, g.s, np.int64), px]).astype(np.int32)
    v = np.concatenate([px, np.full(k, g.t, np.int64)]).astype(np.int32)
    c = np.concatenate([cs, ct]).astype(np.int32)
    return Batch(u, v, c)


# ----------------------------------------------------------------------------
# config 4: unit-capacity bipartite matching
# ----------------------------------------------------------------------------

def bipartite(L: int = 1 << 22, draws: int = 1 << 26, alpha: float = 1.0, seed: int = 4,
              zero_frac: float = 1.0 / 16) -> Graph:
    """Config 4: left ids 0..L-1, right ids L..2L-1, s=2L, t=2L+1.
    `draws` L->R edges: left uniform, right Zipf(alpha) over a random permutation of
    R; duplicates removed; s->l and r->t cap 1; L->R cap 1 except a random
    `zero_frac` that start at 0 (the insert pool)."""
    r = _rng(seed)
    R = L
    lft = r.integers(0, L, size=draws, dtype=np.int64)
    w = 1.0 / np.arange(1, R + 1, dtype=np.float64) ** alpha
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    rank = np.searchsorted(cdf, r.random(draws))
    rank = np.minimum(rank, R - 1)
    perm = r.permutation(R).astype(np.int64)
    rgt = perm[rank]
    key = _unique_sorted(lft * R + rgt)
    lft = key // R
    rgt = key % R + L
    mlr = key.shape[0]
    caplr = np.ones(mlr, np.int32)
    caplr[r.random(mlr) < zero_frac] = 0
    s, t = 2 * L, 2 * L + 1
    u = np.concatenate([np.full(L, s, np.int64), lft, np.arange(L, 2 * L, dtype=np.int64)])
    v = np.concatenate([np.arange(L, dtype=np.int64), rgt, np.full(R, t, np.int64)])
    cap = np.concatenate([np.ones(L, np.int32), caplr, np.ones(R, np.int32)])
    return Graph(2 * L + 2, s, t, u.astype(np.int32), v.astype(np.int32), cap, name=f"bip{L}",
                 meta=dict(L=L, lr_begin=L, lr_end=L + mlr, seed=seed))


def bipartite_batch(g: Graph, st: CapState, frac: float, seed: int) -> Batch:
    """round(frac * |L->R|) L->R edges: half 0->1 inserts, half 1->0 deletes."""
    r = _rng(seed)
    a, b = g.meta["lr_begin"], g.meta["lr_end"]
    u = g.u[a:b]
    v = g.v[a:b]
    cur = st.lookup(u, v)
    k = max(2, int(round(frac * (b - a))))
    zeros = np.nonzero(cur == 0)[0]
    ones = np.nonzero(cur > 0)[0]
    ki = min(k // 2, zeros.shape[0])
    kd = min(k - ki, ones.shape[0])
    pi = r.choice(zeros, size=ki, replace=False) if ki else np.zeros(0, np.int64)
    pd = r.choice(ones, size=kd, replace=False) if kd else np.zeros(0, np.int64)
    idx = np.concatenate([pi, pd])
    new = np.concatenate([np.ones(ki, np.int32), np.zeros(kd, np.int32)])
    return Batch(u[idx].astype(np.int32), v[idx].astype(np.int32), new)


def config_graph(name: str) -> Graph:
    """Named full-size workloads of BASELINE.json's configs."""
    if name == "rmat20":
        return rmat(20, 16, 1, 7)
    if name.startswith("rmat22_"):
        i = int(name.split("_")[1])
        return rmat(22, 16, i, 7)
    if name == "grid2048":
        return grid(2048, 3)
    if name == "bip4m":
        return bipartite()
    raise KeyError(name)


def sequence(spec: dict):
    """(graph, list of batches) of a named cumulative batch sequence, deterministic in
    `spec` (picklable, so that oracle workers can rebuild it):
      {"kind": "rmat", "scale": 20, "seed_graph": 1, "seed_caps": 7, "frac": 0.01,
       "nb": 25, "seed_base": 100}
      {"kind": "grid", "W": 2048, "seed": 3, "frac": 0.01, "nb": 10, "seed_base": 300}
      {"kind": "bip", "L": 2**22, "draws": 2**26, "seed": 4, "frac": 0.01, "nb": 3, "seed_base": 400}
    Batch j is drawn after batches 0..j-1 were applied (cumulative capacities)."""
    kind = spec["kind"]
    if kind == "rmat":
        g = rmat(spec["scale"], spec.get("edge_factor", 16), spec.get("seed_graph", 1), spec.get("seed_caps", 7))
        gen = lambda st, j: rmat_batch(g, st, spec["frac"], spec.get("seed_base", 100) + j)  # noqa: E731
    elif kind == "grid":
        g = grid(spec["W"], spec.get("seed", 3))
        gen = lambda st, j: grid_batch(g, spec["frac"], spec.get("seed_base", 300) + j)  # noqa: E731
    elif kind == "bip":
        g = bipartite(L=spec.get("L", 1 << 22), draws=spec.get("draws", 1 << 26), seed=spec.get("seed", 4))
        gen = lambda st, j: bipartite_batch(g, st, spec["frac"], spec.get("seed_base", 400) + j)  # noqa: E731
    else:
        raise KeyError(kind)
    st = CapState(g)
    out = []
    for j in range(spec["nb"]):
        b = gen(st, j)
        st.apply(b)
        out.append(b)
    if kind == "grid":        # grid_batch drifts the image in g.meta: rebuild it unperturbed
        g = grid(spec["W"], spec.get("seed", 3))
    return g, out
