"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by
element, after the static solve and after EVERY batch.  Integer results, so the
bar is bit-exact: F, S_min (unique minimal source side) and S_max; the exported
device state must also pass the oracle's checker (capacity, pair-sum, excess,
no augmenting path, conversion to a true flow with conservation, cut = F)."""
import numpy as np
import pytest

import oracle as O
import workloads as W
from golden_io import graph, load

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dmf():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2511_05895_b200 as P
    P.load_library()
    return P


def _oracle(g, small=False):
    if small and g.n <= 16:
        b = O.brute_force(g)
        return b["F"], b["smin"], b["smax"]
    r = O.maxflow(g, "dinic")
    return r["F"], r["smin"], r["smax"]


def _verify(f, g, tag, small=False, check=True):
    Fo, smin_o, smax_o = _oracle(g, small)
    F = f.flow_value()
    assert F == Fo, f"{tag}: F gpu={F} oracle={Fo}"
    smin = f.min_cut_source_side()
    assert np.array_equal(smin, smin_o), f"{tag}: S_min differs at {np.nonzero(smin != smin_o)[0][:10]}"
    smax = f.max_cut_source_side()
    assert np.array_equal(smax, smax_o), f"{tag}: S_max differs at {np.nonzero(smax != smax_o)[0][:10]}"
    if check:
        st = f.export_state()
        rc, msg, _ = O.check_state(g.n, g.s, g.t, st["row_ptr"], st["dst"], st["rev"], st["cap"], st["res"], st["e"],
                                   F, smin)
        assert rc == 0, f"{tag}: checker {rc}: {msg}"


@pytest.mark.parametrize("algo", ["pr", "pp"])
def test_clrs_chain(dmf, algo):
    d = load("clrs_26_1.txt")
    g = graph(d)
    f = dmf.DynMaxFlow.from_graph(g)
    assert f.S == 18                        # 9 input edges, 9 distinct pairs -> 9 reverses
    assert f.static_solve() == 23
    _verify(f, g, "clrs static", small=True)
    st = W.CapState(g)
    for j, step in enumerate(d["steps"]):
        b = W.as_batch(step["batch"])
        st.apply(b)
        F = f.apply_batch(b.u, b.v, b.new_cap, algo=algo)
        assert F == step["F"]
        assert np.array_equal(f.min_cut_source_side(), step["smin"])
        _verify(f, st.graph(), f"clrs b{j}", small=True)


@pytest.mark.parametrize("algo", ["pr", "pp"])
def test_spec_g1(dmf, algo):
    d = load("spec_g1.txt")
    g = graph(d)
    for step in d["steps"]:
        f = dmf.DynMaxFlow.from_graph(g)
        assert f.S == 10                    # S:64 "10 slots"
        assert f.static_solve() == 6
        assert np.array_equal(f.min_cut_source_side(), d["smin"])
        assert np.array_equal(f.max_cut_source_side(), d["smax"])
        b = W.as_batch(step["batch"])
        assert f.apply_batch(b.u, b.v, b.new_cap, algo=algo) == step["F"]
        assert np.array_equal(f.min_cut_source_side(), step["smin"])
        assert np.array_equal(f.max_cut_source_side(), step["smax"])
        f.close()


def test_spec_g1_excess_after_update(dmf):
    """after G1's max flow and (0,1)->2 the excess (before repair) is
    [-4,-2,0,6].  With DYN_PR the repair then leaves F = 4."""
    g = graph(load("spec_g1.txt"))
    f = dmf.DynMaxFlow.from_graph(g)
    f.static_solve()
    st = f.export_state()
    assert int(st["e"][3]) == 6 and int(st["e"][0]) == -6
    assert f.apply_batch(np.array([0]), np.array([1]), np.array([2]), algo="pr") == 4


@pytest.mark.parametrize("mode", ["pr", "pp", "mix"])
def test_tiny_random_config1(dmf, mode):
    """Config 1: 200 random graphs (n <= 12) x 10 mixed batches, vs brute force."""
    rng = np.random.default_rng(5)
    for seed in range(200):
        g = W.tiny_random(seed)
        f = dmf.DynMaxFlow.from_graph(g)
        f.static_solve()
        _verify(f, g, f"tiny{seed} static", small=True, check=seed % 10 == 0)
        st = W.CapState(g)
        for j, b in enumerate(W.tiny_batches(g, seed)):
            st.apply(b)
            algo = mode if mode != "mix" else ("pr" if rng.random() < 0.5 else "pp")
            f.apply_batch(b.u, b.v, b.new_cap, algo=algo)
            _verify(f, st.graph(), f"tiny{seed} b{j} {algo}", small=True, check=seed % 10 == 0)
        f.close()


@pytest.mark.parametrize("scale,algo", [(12, "pr"), (12, "pp"), (15, "pp"), (15, "pr")])
def test_rmat_medium(dmf, scale, algo):
    g = W.rmat(scale, 16, 1, 7)
    f = dmf.DynMaxFlow.from_graph(g)
    f.static_solve()
    _verify(f, g, f"rmat{scale} static")
    st = W.CapState(g)
    for j, frac in enumerate([0.001, 0.01, 0.1, 0.01, 0.001]):
        b = W.rmat_batch(g, st, frac, 100 + j)
        st.apply(b)
        f.apply_batch(b.u, b.v, b.new_cap, algo=algo)
        _verify(f, st.graph(), f"rmat{scale} b{j} {algo}")


@pytest.mark.parametrize("algo", ["pr", "pp"])
def test_grid_medium(dmf, algo):
    g = W.grid(128, 3)
    f = dmf.DynMaxFlow.from_graph(g)
    f.static_solve()
    _verify(f, g, "grid static")
    st = W.CapState(g)
    for j, frac in enumerate([0.001, 0.01, 0.1]):
        b = W.grid_batch(g, frac, 300 + j)
        st.apply(b)
        f.apply_batch(b.u, b.v, b.new_cap, algo=algo)
        _verify(f, st.graph(), f"grid b{j} {algo}")


@pytest.mark.parametrize("algo", ["pr", "pp"])
def test_bipartite_medium(dmf, algo):
    g = W.bipartite(L=1 << 12, draws=1 << 16, seed=4)
    f = dmf.DynMaxFlow.from_graph(g)
    F0 = f.static_solve()
    L = g.meta["L"]
    a, b_ = g.meta["lr_begin"], g.meta["lr_end"]
    lr = g.cap[a:b_] > 0
    assert F0 == O.hopcroft_karp(L, L, g.u[a:b_][lr], g.v[a:b_][lr] - L)
    _verify(f, g, "bip static")
    st = W.CapState(g)
    for j, frac in enumerate([0.001, 0.01, 0.1]):
        b = W.bipartite_batch(g, st, frac, 400 + j)
        st.apply(b)
        f.apply_batch(b.u, b.v, b.new_cap, algo=algo)
        _verify(f, st.graph(), f"bip b{j} {algo}")


def test_terminal_only_grid_closed_form(dmf):
    g = W.grid(256, 11, nlinks=False)
    npx = 256 * 256
    F, side = O.grid_terminal_closed_form(g.cap[:npx], g.cap[npx:2 * npx])
    f = dmf.DynMaxFlow.from_graph(g)
    assert f.static_solve() == F
    want = np.zeros(g.n, np.uint8)
    want[:npx] = side
    want[g.s] = 1
    assert np.array_equal(f.min_cut_source_side(), want)


# ------------------------------------------------------------------ boundary behaviour

def test_create_merges_duplicates_and_rejects_bad_input(dmf):
    # duplicates (0,1) merged by summing: single slot of cap 5 + its reverse
    row_ptr = np.array([0, 2, 2, 2], np.int64)
    f = dmf.DynMaxFlow(3, row_ptr, np.array([1, 1], np.int32), np.array([2, 3], np.int32), 0, 1)
    assert f.S == 2 and f.m == 1
    assert f.static_solve() == 5
    for col, cap, s, t in [([0], [1], 0, 1), ([5], [1], 0, 1), ([1], [-1], 0, 1), ([1], [1], 0, 0)]:
        with pytest.raises(dmf.DMFError) as ei:
            dmf.DynMaxFlow(3, np.array([0, 1, 1, 1], np.int64), np.array(col, np.int32), np.array(cap, np.int32), s, t)
        assert ei.value.code == -1
    with pytest.raises(dmf.DMFError) as ei:
        dmf.DynMaxFlow(3, np.array([0, 2, 2, 2], np.int64), np.array([1, 1], np.int32),
                       np.array([dmf.CAP_MAX, 5], np.int32), 0, 1)
    assert ei.value.code == -7


def test_batch_errors_leave_state_unchanged(dmf):
    g = W.rmat(10, 8, 2, 3)
    f = dmf.DynMaxFlow.from_graph(g)
    with pytest.raises(dmf.DMFError) as ei:            # PP before any solve
        f.apply_batch(g.u[:1], g.v[:1], g.cap[:1], algo="pp")
    assert ei.value.code == -4
    F0 = f.static_solve()
    before = f.export_state()
    bad = [
        ((g.u[:3], g.v[:3], np.array([1, 2, 3])), None),
        ((np.array([g.u[0], g.u[0]]), np.array([g.v[0], g.v[0]]), np.array([1, 2])), -3),   # duplicate
        ((np.array([0]), np.array([0]), np.array([1])), -2),                                   # self-loop: no slot
        ((np.array([g.n]), np.array([0]), np.array([1])), -1),                                 # out of range
        ((g.u[:1], g.v[:1], np.array([-1])), -7),                                              # negative cap
        ((g.u[:1], g.v[:1], np.array([dmf.CAP_MAX + 1], np.int64)), -7),
    ]
    # a pair that is neither an edge nor a reverse
    keys = set(zip(g.u.tolist(), g.v.tolist())) | set(zip(g.v.tolist(), g.u.tolist()))
    a = next((x, y) for x in range(g.n) for y in range(g.n) if x != y and (x, y) not in keys)
    bad.append(((np.array([a[0]]), np.array([a[1]]), np.array([5])), -2))
    for (u, v, c), code in bad[1:]:
        c = np.asarray(c).astype(np.int64).clip(-2**31, 2**31 - 1).astype(np.int32)
        for algo in ("pr", "pp"):
            with pytest.raises(dmf.DMFError) as ei:
                f.apply_batch(np.asarray(u, np.int32), np.asarray(v, np.int32), c, algo=algo)
            assert ei.value.code == code
            after = f.export_state()
            for k in before:
                assert np.array_equal(before[k], after[k]), k
            assert f.flow_value() == F0
    # an empty batch is a fixed point
    assert f.apply_batch(np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros(0, np.int32), algo="pr") == F0
    assert f.apply_batch(np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros(0, np.int32), algo="pp") == F0


def test_device_pointer_batches(dmf):
    import torch
    g = W.rmat(12, 8, 4, 5)
    f = dmf.DynMaxFlow.from_graph(g)
    f.static_solve()
    st = W.CapState(g)
    b = W.rmat_batch(g, st, 0.05, 9)
    st.apply(b)
    tu = torch.from_numpy(b.u).cuda()
    tv = torch.from_numpy(b.v).cuda()
    tc = torch.from_numpy(b.new_cap).cuda()
    f.apply_batch(tu, tv, tc, algo="pp")
    mask = torch.zeros(g.n, dtype=torch.uint8, device="cuda")
    f.min_cut_source_side(mask)
    Fo, smin, _ = _oracle(st.graph())
    assert f.flow_value() == Fo
    assert np.array_equal(mask.cpu().numpy(), smin)


def test_static_resolve_after_batches_matches(dmf):
    """A static re-solve on the updated capacities (the paper's baseline)
    gives the same F and cuts as the dynamic repair."""
    g = W.rmat(13, 16, 1, 7)
    f = dmf.DynMaxFlow.from_graph(g)
    f.static_solve()
    st = W.CapState(g)
    for j in range(3):
        b = W.rmat_batch(g, st, 0.01, 700 + j)
        st.apply(b)
        Fd = f.apply_batch(b.u, b.v, b.new_cap, algo="pp")
        mask_d = f.min_cut_source_side()
        Fs = f.static_solve()
        assert Fs == Fd
        assert np.array_equal(f.min_cut_source_side(), mask_d)


# ------------------------------------------------------------------ static push-pull

def test_static_pp_tiny_random(dmf):
    """dmf_static_solve_pp on 200 random graphs (n <= 12) vs brute force,
    then one mixed PP batch each."""
    for seed in range(200):
        g = W.tiny_random(seed)
        f = dmf.DynMaxFlow.from_graph(g)
        f.static_solve_pp()
        _verify(f, g, f"tiny{seed} static-pp", small=True)
        st = W.CapState(g)
        for j, b in enumerate(W.tiny_batches(g, seed, nb=2)):
            st.apply(b)
            f.apply_batch(b.u, b.v, b.new_cap, algo="pp")
            _verify(f, st.graph(), f"tiny{seed} pp b{j} after static-pp", small=True)
        f.close()


@pytest.mark.parametrize("name", ["clrs", "rmat13", "grid"])
def test_static_pp_matches(dmf, name):
    """Static push-pull gives the static solve's F / S_min / S_max (and passes the
    checker); PP batches continue exactly from its partition."""
    if name == "clrs":
        g = graph(load("clrs_26_1.txt"))
    elif name == "rmat13":
        g = W.rmat(13, 16, 1, 7)
    else:
        g = W.grid(96, 3)
    f = dmf.DynMaxFlow.from_graph(g)
    f.static_solve_pp()
    _verify(f, g, f"{name} static-pp", small=(name == "clrs"))
    if name == "rmat13":
        st = W.CapState(g)
        for j in range(2):
            b = W.rmat_batch(g, st, 0.01, 950 + j)
            st.apply(b)
            f.apply_batch(b.u, b.v, b.new_cap, algo="pp")
            _verify(f, st.graph(), f"{name} pp b{j} after static-pp")
    f.close()


# ------------------------------------------------------------------ stage (ii): true flow

def _assert_true_flow(f, g, F, tag):
    """The exported state is a feasible maximum flow of value F: e(v) = 0 off {s,t},
    e(t) = -e(s) = F, 0 <= res <= cap + cap_rev, net outflow of every vertex = -e(v)
    (conservation), and dmf_edge_flow = max(0, cap - res) within [0, cap]."""
    st = f.export_state()
    e, rp, res, cap, rev = st["e"], st["row_ptr"], st["res"], st["cap"], st["rev"]
    off = np.ones(g.n, bool); off[[g.s, g.t]] = False
    assert not e[off].any(), f"{tag}: {int((e[off] != 0).sum())} vertices keep excess/deficit"
    assert e[g.t] == F and e[g.s] == -F, f"{tag}: e(t)={e[g.t]} e(s)={e[g.s]} F={F}"
    assert (res >= 0).all() and (res <= cap.astype(np.int64) + cap[rev]).all(), f"{tag}: capacity"
    src = np.repeat(np.arange(g.n), np.diff(rp))
    net = np.bincount(src, weights=(cap.astype(np.int64) - res), minlength=g.n)
    assert np.array_equal(net.astype(np.int64), -e), f"{tag}: conservation"
    fl = f.edge_flow()
    assert np.array_equal(fl, np.maximum(cap - res, 0)) and (fl <= cap).all(), f"{tag}: edge flow"
    assert not ((fl > 0) & (fl[rev] > 0)).any(), f"{tag}: both directions of a pair carry flow"


@pytest.mark.parametrize("algo", ["pr", "pp"])
def test_to_flow_clrs_chain(dmf, algo):
    """dmf_to_flow after every CLRS batch (decrements below the flow leave deficits
    that must be filled from t): a true flow, F / S_min unchanged, later batches exact."""
    d = load("clrs_26_1.txt")
    g = graph(d)
    f = dmf.DynMaxFlow.from_graph(g)
    f.static_solve()
    st = W.CapState(g)
    for j, step in enumerate(d["steps"]):
        bb = W.as_batch(step["batch"])
        st.apply(bb)
        f.apply_batch(bb.u, bb.v, bb.new_cap, algo=algo)
        F, smin = f.flow_value(), f.min_cut_source_side()
        assert f.to_flow() == F == step["F"]
        assert np.array_equal(f.min_cut_source_side(), smin)
        _assert_true_flow(f, st.graph(), F, f"clrs b{j} {algo}")
    f.close()


@pytest.mark.parametrize("scale,algo", [(12, "pp"), (14, "pr"), (14, "pp")])
def test_to_flow_rmat(dmf, scale, algo):
    """Stage (ii) on RMAT after static + mixed batches, then more batches on the
    converted state: F, S_min and S_max stay bit-exact with the oracle."""
    g = W.rmat(scale, 16, 1, 7)
    f = dmf.DynMaxFlow.from_graph(g)
    f.static_solve()
    st = W.CapState(g)
    for j in range(4):
        b = W.rmat_batch(g, st, 0.01, 900 + j)
        st.apply(b)
        f.apply_batch(b.u, b.v, b.new_cap, algo=algo)
        if j % 2 == 0:
            F = f.flow_value()
            assert f.to_flow() == F
            _assert_true_flow(f, st.graph(), F, f"rmat{scale} b{j} {algo}")
        _verify(f, st.graph(), f"rmat{scale} b{j} {algo} (after stage ii)")
    f.close()


# ------------------------------------------------------------------ full-size configs
# BASELINE.json configs 2-5 at full size, in the launch configuration bench.py times
# (default grid, KERNELCYCLES = floor(m/n), default knobs).  F and S_min are compared
# bit-exactly with the oracle (two-phase FIFO push-relabel, a full recompute per
# batch on a pool of worker processes: oracle/pool.py) after the static solve and
# after EVERY batch.

def _replay(dmf, spec, algos, check_at=(), knobs=None):
    """Static solve + the batches of `spec` on one handle; returns per-batch (F, S_min)
    (index -1 = after the static solve) and the handle."""
    g, batches = W.sequence(spec)
    f = dmf.DynMaxFlow.from_graph(g, **(knobs or {}))
    f.static_solve()
    got = {-1: (f.flow_value(), f.min_cut_source_side().copy())}
    for j, b in enumerate(batches):
        f.apply_batch(b.u, b.v, b.new_cap, algo=algos[j % len(algos)])
        got[j] = (f.flow_value(), f.min_cut_source_side().copy())
        if j in check_at:
            st = W.CapState(g)
            for bb in batches[:j + 1]:
                st.apply(bb)
            gg = st.graph()
            stt = f.export_state()
            rc, msg, _ = O.check_state(gg.n, gg.s, gg.t, stt["row_ptr"], stt["dst"], stt["rev"], stt["cap"],
                                       stt["res"], stt["e"], got[j][0], got[j][1])
            assert rc == 0, f"b{j}: checker {rc}: {msg}"
    return got, f


def _compare(spec, got, tag):
    from oracle.pool import recompute
    res = recompute(spec, sorted(got))
    assert len(res) == len(got), f"{tag}: oracle finished {len(res)} of {len(got)} recomputes"
    for r in res:
        F, smin = got[r["j"]]
        assert F == r["F"], f"{tag} b{r['j']}: F gpu={F} oracle={r['F']}"
        assert np.array_equal(smin, r["smin"]), \
            f"{tag} b{r['j']}: S_min differs ({int((smin != r['smin']).sum())} vertices)"


@pytest.mark.full
@pytest.mark.parametrize("workload", ["rmat22", "rmat20"])
def test_bench_sequence_full(dmf, workload):
    """EXACTLY the batches bench.py times (its workload spec, warm-up + timed steps), in
    its launch configuration, DYN_PP, checked after every batch."""
    import bench
    spec = bench.workload_spec(workload, bench.DEFAULT_WARMUP, bench.DEFAULT_STEPS)
    got, f = _replay(dmf, spec, ["pp"], check_at=(0,))
    f.close()
    _compare(spec, got, workload)


@pytest.mark.full
def test_config2_rmat20_mixed_fractions_full(dmf):
    """Config 2: RMAT-20 (1M / 16.1M), 1% / 0.1% / 10% mixed batches, PP and PR interleaved."""
    specs = [dict(kind="rmat", scale=20, frac=fr, nb=3, seed_base=100 + 10 * i) for i, fr in enumerate([0.001, 0.1])]
    for spec in specs:
        got, f = _replay(dmf, spec, ["pr", "pp"], check_at=(1,))
        f.close()
        _compare(spec, got, f"rmat20 frac {spec['frac']}")


@pytest.mark.full
def test_config3_grid2048_full(dmf):
    """Config 3: 2048x2048 segmentation grid, 10 terminal-capacity batches (1% of pixels),
    PR and PP interleaved."""
    spec = dict(kind="grid", W=2048, seed=3, frac=0.01, nb=10, seed_base=300)
    got, f = _replay(dmf, spec, ["pr", "pp"], check_at=(3,))
    f.close()
    _compare(spec, got, "grid2048")


@pytest.mark.full
@pytest.mark.parametrize("algo", ["pp", "pr"])
def test_config4_bipartite_full(dmf, algo):
    """Config 4: unit bipartite 4M+4M / 72.7M merged edges; static F = Hopcroft-Karp
    matching; 3 cumulative 1% insert/delete batches under PR and under PP."""
    spec = dict(kind="bip", frac=0.01, nb=3, seed_base=400)
    g, _ = W.sequence(dict(spec, nb=0))
    L = g.meta["L"]
    a, b_ = g.meta["lr_begin"], g.meta["lr_end"]
    lr = g.cap[a:b_] > 0
    got, f = _replay(dmf, spec, [algo])
    f.close()
    assert got[-1][0] == O.hopcroft_karp(L, L, g.u[a:b_][lr], g.v[a:b_][lr] - L)
    del got[-1]
    _compare(spec, got, f"bip {algo}")


@pytest.mark.full
def test_config5_rmat22_snapshots_full(dmf):
    """Config 5: two more RMAT-22 snapshots (graph seeds 2 and 3), 3 PP batches each."""
    for seed in (2, 3):
        spec = dict(kind="rmat", scale=22, seed_graph=seed, frac=0.01, nb=3, seed_base=100)
        got, f = _replay(dmf, spec, ["pp"])
        f.close()
        _compare(spec, got, f"rmat22 seed {seed}")
