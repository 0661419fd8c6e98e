"""Pins for the CPU oracle (-m "not gpu").  Each test ties an oracle function to
something other than itself: a textbook / paper worked example (tests/golden),
brute-force cut enumeration, a closed form, an independent library (scipy),
Hopcroft-Karp, or weak duality (feasible flow value == cut capacity)."""
import numpy as np
import pytest

import oracle as O
import workloads as W
from golden_io import graph, load
from slotform import slots, state_from_flow

ALGOS = ["ek", "dinic", "fifo_pr"]


def _check_flow_feasible(g, flow, F):
    """Capacity and conservation of a per-edge flow, value F (definition)."""
    assert np.all(flow >= 0) and np.all(flow <= g.cap)
    net = np.zeros(g.n, np.int64)
    np.add.at(net, g.v, flow)
    np.add.at(net, g.u, -flow)
    for x in range(g.n):
        if x not in (g.s, g.t):
            assert net[x] == 0
    assert net[g.t] == F and net[g.s] == -F


def _cut_capacity(g, side):
    m = side.astype(bool)
    return int(g.cap[m[g.u] & ~m[g.v]].astype(np.int64).sum())


# ------------------------------------------------------------------ golden examples

@pytest.mark.parametrize("algo", ALGOS)
def test_clrs_26_1_and_chain(algo):
    d = load("clrs_26_1.txt")
    g = graph(d)
    r = O.maxflow(g, algo)
    assert r["F"] == d["F"] == 23
    assert np.array_equal(r["smin"], d["smin"]) and np.array_equal(r["smax"], d["smax"])
    st = W.CapState(g)
    for step in d["steps"]:
        st.apply(W.as_batch(step["batch"]))
        r = O.maxflow(st.graph(), algo)
        assert r["F"] == step["F"]
        assert np.array_equal(r["smin"], step["smin"]) and np.array_equal(r["smax"], step["smax"])


@pytest.mark.parametrize("algo", ALGOS)
def test_spec_g1(algo):
    d = load("spec_g1.txt")
    g = graph(d)
    r = O.maxflow(g, algo)
    assert r["F"] == 6
    assert np.array_equal(r["smin"], d["smin"]) and np.array_equal(r["smax"], d["smax"])
    for step in d["steps"]:
        st = W.CapState(g)          # every G1 batch applies to the original G1
        st.apply(W.as_batch(step["batch"]))
        r = O.maxflow(st.graph(), algo)
        assert r["F"] == step["F"]
        assert np.array_equal(r["smin"], step["smin"]) and np.array_equal(r["smax"], step["smax"])


def test_brute_force_golden():
    for name in ("clrs_26_1.txt", "spec_g1.txt"):
        d = load(name)
        b = O.brute_force(graph(d))
        assert b["F"] == d["F"]
        assert np.array_equal(b["smin"], d["smin"]) and np.array_equal(b["smax"], d["smax"])


# ------------------------------------------------------------------ special cases

@pytest.mark.parametrize("algo", ALGOS)
def test_single_edge_and_no_path(algo):
    g = W.Graph(2, 0, 1, np.array([0], np.int32), np.array([1], np.int32), np.array([7], np.int32))
    r = O.maxflow(g, algo)
    assert r["F"] == 7 and list(r["smin"]) == [1, 0]
    # no s-t path: F = 0 and S_min = s's reach
    g = W.Graph(4, 0, 3, np.array([0, 1, 3], np.int32), np.array([1, 2, 2], np.int32), np.array([5, 5, 5], np.int32))
    r = O.maxflow(g, algo)
    assert r["F"] == 0 and list(r["smin"]) == [1, 1, 1, 0]
    # parallel edges are summed; self-loops carry nothing
    g = W.Graph(3, 0, 2, np.array([0, 0, 1, 1], np.int32), np.array([1, 1, 2, 1], np.int32), np.array([2, 3, 9, 4], np.int32))
    assert O.maxflow(g, algo)["F"] == 5


# ------------------------------------------------------------------ brute force (config 1)

def test_tiny_random_vs_brute_force():
    """Config 1: 200 random graphs (n <= 12) x 10 cumulative mixed batches; all
    three algorithms equal brute-force cut enumeration on F, S_min and S_max."""
    nstates = 0
    for seed in range(200):
        g = W.tiny_random(seed)
        st = W.CapState(g)
        batches = W.tiny_batches(g, seed)
        for j in range(len(batches) + 1):
            if j:
                st.apply(batches[j - 1])
            cur = st.graph()
            b = O.brute_force(cur)
            for algo in ALGOS:
                r = O.maxflow(cur, algo, want_flow=True)
                assert r["F"] == b["F"], (seed, j, algo)
                assert np.array_equal(r["smin"], b["smin"]), (seed, j, algo)
                assert np.array_equal(r["smax"], b["smax"]), (seed, j, algo)
                _check_flow_feasible(cur, r["flow"], r["F"])
            nstates += 1
    assert nstates == 2200


# ------------------------------------------------------------------ independent library

def _scipy_F(g):
    import scipy.sparse as sp
    from scipy.sparse.csgraph import maximum_flow
    keep = g.u != g.v
    A = sp.coo_matrix((g.cap[keep].astype(np.int32), (g.u[keep], g.v[keep])), shape=(g.n, g.n)).tocsr()
    A.sum_duplicates()
    return int(maximum_flow(A, g.s, g.t, method="dinic").flow_value)


@pytest.mark.parametrize("scale", [10, 13])
def test_rmat_vs_scipy_and_duality(scale):
    g = W.rmat(scale, 16, 1, 7)
    Fs = _scipy_F(g)
    for algo in (["ek"] if scale <= 10 else []) + ["dinic", "fifo_pr"]:
        r = O.maxflow(g, algo, want_flow=True)
        assert r["F"] == Fs
        _check_flow_feasible(g, r["flow"], r["F"])
        # weak duality certificate: a feasible flow of value F and a cut of capacity F
        assert _cut_capacity(g, r["smin"]) == r["F"]
        assert _cut_capacity(g, r["smax"]) == r["F"]
        assert r["smin"][g.s] == 1 and r["smin"][g.t] == 0
        assert np.all(r["smin"] <= r["smax"])


def test_grid_with_nlinks_vs_scipy():
    g = W.grid(64, 5)
    Fs = _scipy_F(g)
    for algo in ["dinic", "fifo_pr"]:
        r = O.maxflow(g, algo, want_flow=True)
        assert r["F"] == Fs
        _check_flow_feasible(g, r["flow"], r["F"])
        assert _cut_capacity(g, r["smin"]) == r["F"]


# ------------------------------------------------------------------ closed forms

@pytest.mark.parametrize("algo", ["dinic", "fifo_pr"])
def test_terminal_only_grid_closed_form(algo):
    g = W.grid(96, 11, nlinks=False)
    npx = 96 * 96
    cs = g.cap[:npx]
    ct = g.cap[npx:2 * npx]
    F, side = O.grid_terminal_closed_form(cs, ct)
    r = O.maxflow(g, algo)
    assert r["F"] == F
    want = np.zeros(g.n, np.uint8)
    want[:npx] = side
    want[g.s] = 1
    assert np.array_equal(r["smin"], want)


def test_bipartite_hopcroft_karp():
    g = W.bipartite(L=1 << 11, draws=1 << 14, seed=4)
    L = g.meta["L"]
    a, b = g.meta["lr_begin"], g.meta["lr_end"]
    lr = g.cap[a:b] > 0
    M = O.hopcroft_karp(L, L, g.u[a:b][lr], g.v[a:b][lr] - L)
    for algo in ["dinic", "fifo_pr"]:
        assert O.maxflow(g, algo)["F"] == M
    # HK itself on a hand example: a 3x3 bipartite graph whose maximum matching is 2
    assert O.hopcroft_karp(3, 3, np.array([0, 1, 2]), np.array([0, 0, 1])) == 2
    assert O.hopcroft_karp(3, 3, np.array([0, 0, 1, 2]), np.array([0, 1, 0, 2])) == 3


def test_monotonicity_under_batches():
    """inc-only batches never decrease F, dec-only never increase it, |dF| <= sum|dc|."""
    g = W.rmat(10, 8, 3, 9, capmax=100)
    st = W.CapState(g)
    F0 = O.maxflow(g, "dinic")["F"]
    for j, kind in enumerate(["inc", "dec", "inc", "dec"]):
        b = W.rmat_batch(g, st, 0.05, 200 + j, kind=kind, capmax=100)
        dc = int(np.abs(b.new_cap.astype(np.int64) - st.lookup(b.u, b.v)).sum())
        st.apply(b)
        F1 = O.maxflow(st.graph(), "dinic")["F"]
        assert (F1 >= F0) if kind == "inc" else (F1 <= F0)
        assert abs(F1 - F0) <= dc
        F0 = F1


# ------------------------------------------------------------------ checker pins

def _g1():
    return [(0, 1, 4), (0, 2, 2), (1, 2, 3), (1, 3, 1), (2, 3, 6)]


def test_checker_accepts_true_max_flow_g1():
    # max flow of G1 (F=6): 0->1:4, 0->2:2, 1->3:1, 1->2:3, 2->3:5
    st = state_from_flow(4, _g1(), {(0, 1): 4, (0, 2): 2, (1, 3): 1, (1, 2): 3, (2, 3): 5})
    rc, msg, _ = O.check_state(4, 0, 3, *st, F=6, smin=np.array([1, 0, 0, 0], np.uint8))
    assert rc == 0, msg


def test_checker_accepts_converged_pseudoflow_with_deficit():
    # G1 at max flow then (0,1)->2 with the Alg.5 clamp: flow on (0,1)
    # drops to 2, excess becomes [-4,-2,0,6]; nothing can be augmented, F = 6-2 = 4.
    edges = [(0, 1, 2), (0, 2, 2), (1, 2, 3), (1, 3, 1), (2, 3, 6)]
    st = state_from_flow(4, edges, {(0, 1): 2, (0, 2): 2, (1, 3): 1, (1, 2): 3, (2, 3): 5})
    assert list(st[5]) == [-4, -2, 0, 6]          # S:84 "excess = [-4,-2,0,6]"
    rc, msg, _ = O.check_state(4, 0, 3, *st, F=4, smin=np.array([1, 0, 0, 0], np.uint8))
    assert rc == 0, msg


def test_checker_rejects_tampering():
    good = state_from_flow(4, _g1(), {(0, 1): 4, (0, 2): 2, (1, 3): 1, (1, 2): 3, (2, 3): 5})
    smin = np.array([1, 0, 0, 0], np.uint8)
    row_ptr, dst, rev, cap, res, e = good
    assert O.check_state(4, 0, 3, *good, F=7, smin=smin)[0] == 7            # wrong F
    assert O.check_state(4, 0, 3, *good, F=6, smin=np.array([1, 1, 0, 0], np.uint8))[0] == 8
    r2 = res.copy(); r2[rev[0]] -= 1     # slot (1,0) holds 4: still in range, pair-sum broken
    assert O.check_state(4, 0, 3, row_ptr, dst, rev, cap, r2, e, F=6, smin=smin)[0] == 3
    r3 = res.copy(); r3[0] = -1; r3[rev[0]] += 1 + res[0]
    assert O.check_state(4, 0, 3, row_ptr, dst, rev, cap, r3, e, F=6, smin=smin)[0] == 2
    e2 = e.copy(); e2[1] += 1; e2[2] -= 1
    assert O.check_state(4, 0, 3, row_ptr, dst, rev, cap, res, e2, F=6, smin=smin)[0] == 4
    # SPEC S:202 init_preflow state of G1: e=[-6,4,2,0] -> an augmenting path exists
    pre = state_from_flow(4, _g1(), {(0, 1): 4, (0, 2): 2})
    assert list(pre[5]) == [-6, 4, 2, 0]
    assert O.check_state(4, 0, 3, *pre, F=0, smin=None)[0] == 5
    rv = rev.copy(); rv[0], rv[1] = rv[1], rv[0]
    assert O.check_state(4, 0, 3, row_ptr, dst, rv, cap, res, e, F=6, smin=smin)[0] == 1


def test_slot_counts_g1():
    # G1 has 10 slots (5 original + 5 zero-capacity reverses)
    row_ptr, dst, rev, cap, _ = slots(4, _g1())
    assert len(dst) == 10 and int(cap.sum()) == 16
    assert np.all(rev[rev] == np.arange(10))
