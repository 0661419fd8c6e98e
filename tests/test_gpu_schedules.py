"""GPU parity of every work schedule and every path that only a knob or a failure
reaches.  None of the dmf_options knobs may change a result (F, S_min and S_max are
unique), so each schedule is compared bit-exactly with brute force / Dinic after the
static solve and after EVERY batch, and the exported state must pass the oracle's
checker.  Covered here:

* the schedules of dmf_options.schedule: ASYNC ring, ROUNDS, TOPOLOGY-driven (SURVEY
  N1) and the auto-switch between worklist and topology;
* the local gap exit (R14 form 2) on and off, the DYN_PP warm start on and off;
* forced budget stops (budget_mul < 0) and forced progress stops of the ASYNC tail
  (tail_items = 1): the sweep path that hands queued work to the next global relabel;
* DMF_ENOCONV (max_iters = 1) leaves a valid, unconverged handle;
* checkpoint export -> dmf_import_state -> DYN_PR repair, and check_level = 1;
* device-pointer batches and masks on torch's default stream (no implicit syncs).
"""
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


def _oracle(g):
    if g.n <= 16:
        b = O.brute_force(g)
        return b["F"], b["smin"], b["smax"]
    r = O.maxflow(g, "dinic")
    return r["F"], r["smin"], r["smax"]


def _verify(f, g, tag, check=True):
    Fo, smin_o, smax_o = _oracle(g)
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


KNOB_SETS = {
    "async": dict(schedule="async"),
    "rounds": dict(schedule="rounds"),
    "topology": dict(schedule="topology"),
    "auto_topo_switch": dict(schedule="auto", topo_div=1000000),     # any active vertex -> topology phase
    "auto_topo_n16": dict(topo_div=16),
    "no_gap": dict(local_gap=-1),
    "no_warm": dict(warm=-1),
    "no_certify": dict(certify=-1),
    "budget_stop_async": dict(schedule="async", budget_mul=-1000000, tail_items=1),
    "budget_stop_rounds": dict(schedule="rounds", budget_mul=-1000000),
    "budget_stop_topology": dict(schedule="topology", budget_mul=-1000000),
}


@pytest.mark.parametrize("name", list(KNOB_SETS))
def test_tiny_random_every_schedule(dmf, name):
    """Config 1 (n <= 12, 10 mixed batches) under every knob set, PR / PP mixed, vs brute force."""
    knobs = KNOB_SETS[name]
    rng = np.random.default_rng(11)
    for seed in range(0, 200, 4):
        g = W.tiny_random(seed)
        f = dmf.DynMaxFlow.from_graph(g, **knobs)
        f.static_solve()
        _verify(f, g, f"{name} tiny{seed} static", check=seed % 20 == 0)
        st = W.CapState(g)
        for j, b in enumerate(W.tiny_batches(g, seed)):
            st.apply(b)
            algo = "pr" if rng.random() < 0.4 else "pp"
            f.apply_batch(b.u, b.v, b.new_cap, algo=algo)
            _verify(f, st.graph(), f"{name} tiny{seed} b{j} {algo}", check=seed % 20 == 0)
        f.close()


@pytest.mark.parametrize("name", list(KNOB_SETS))
@pytest.mark.parametrize("algo", ["pp", "pr"])
def test_rmat15_every_schedule(dmf, name, algo):
    """RMAT-15 (32k / 0.5M), 1% / 0.1% / 10% mixed batches under every knob set, vs Dinic
    + the checker; the stats show the knob's path was taken."""
    knobs = KNOB_SETS[name]
    g = W.rmat(15, 16, 1, 7)
    f = dmf.DynMaxFlow.from_graph(g, **knobs)
    f.static_solve()
    # (the static solve counts: from zero flow it is where n/16 vertices are active at once)
    seen = {k: f.stats()[k] for k in ("topology_rounds", "budget_stops", "tail_stops", "rounds")}
    _verify(f, g, f"{name} rmat15 static")
    st = W.CapState(g)
    for j, frac in enumerate([0.01, 0.001, 0.1, 0.01]):
        b = W.rmat_batch(g, st, frac, 100 + j)
        st.apply(b)
        f.apply_batch(b.u, b.v, b.new_cap, algo=algo)
        s = f.stats()
        for k in seen:
            seen[k] += s[k]
        _verify(f, st.graph(), f"{name} rmat15 b{j} {algo}", check=j % 2 == 0)
    # forced topology phases must show up; the realistic n/16 threshold may or may not
    # fire on this graph (it is there for parity of whatever mix of phases it picks)
    if knobs.get("schedule") == "topology" or knobs.get("topo_div", 0) >= 1000000:
        assert seen["topology_rounds"] > 0
    if "budget_mul" in knobs:
        assert seen["budget_stops"] + seen["tail_stops"] > 0
    f.close()


@pytest.mark.parametrize("name", ["async", "rounds", "topology", "no_gap"])
def test_grid_and_bipartite_schedules(dmf, name):
    """Grid 96^2 and unit bipartite 2^11 under the main schedules (vs Dinic / Hopcroft-Karp)."""
    knobs = KNOB_SETS[name]
    for g, gen in ((W.grid(96, 3), lambda g, st, j: W.grid_batch(g, 0.01, 300 + j)),
                   (W.bipartite(L=1 << 11, draws=1 << 15, seed=4), lambda g, st, j: W.bipartite_batch(g, st, 0.01, 400 + j))):
        f = dmf.DynMaxFlow.from_graph(g, **knobs)
        f.static_solve()
        _verify(f, g, f"{name} {g.name} static")
        st = W.CapState(g)
        for j in range(3):
            b = gen(g, st, j)
            st.apply(b)
            f.apply_batch(b.u, b.v, b.new_cap, algo="pp" if j != 1 else "pr")
            _verify(f, st.graph(), f"{name} {g.name} b{j}", check=j == 0)
        f.close()


def test_local_gap_fires_and_is_result_neutral(dmf):
    """The local gap exit is actually exercised (levels found empty, discharges parked)
    -- an asynchronous static solve and PP batches on RMAT-12/13 -- and changes nothing
    in F / S_min / S_max."""
    fired = 0
    for scale in (12, 13):
        g = W.rmat(scale, 16, 1, 7)
        res = {}
        for gap in (0, -1):
            f = dmf.DynMaxFlow.from_graph(g, local_gap=gap, schedule="async")
            f.static_solve()
            s = f.stats()
            out = [(f.flow_value(), f.min_cut_source_side().copy(), f.max_cut_source_side().copy())]
            lv, sk = s["gap_levels"], s["gap_skips"]
            st = W.CapState(g)
            for j in range(4):
                b = W.rmat_batch(g, st, 0.01, 800 + j)
                st.apply(b)
                f.apply_batch(b.u, b.v, b.new_cap, algo="pp")
                s = f.stats()
                lv += s["gap_levels"]; sk += s["gap_skips"]
                out.append((f.flow_value(), f.min_cut_source_side().copy(), f.max_cut_source_side().copy()))
            res[gap] = (out, lv, sk)
            f.close()
        for a, b in zip(res[0][0], res[-1][0]):
            assert a[0] == b[0] and np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])
        assert res[-1][1] == 0 and res[-1][2] == 0
        fired += res[0][1]
    assert fired > 0, "no emptied level was detected"


# ------------------------------------------------------------------ failure / state paths

def test_enoconv_leaves_a_valid_unconverged_handle(dmf):
    """max_iters = 1 forces DMF_ENOCONV; the handle then refuses flow / cut queries and
    DYN_PP (DMF_ESTATE) until a DYN_PR repair converges from the valid pseudoflow."""
    g = W.rmat(12, 16, 1, 7)
    f = dmf.DynMaxFlow.from_graph(g, max_iters=1)
    with pytest.raises(dmf.DMFError) as ei:
        f.static_solve()
    assert ei.value.code == -8
    for call in (f.flow_value, f.min_cut_source_side, lambda: f.apply_batch(g.u[:1], g.v[:1], g.cap[:1], algo="pp")):
        with pytest.raises(dmf.DMFError) as ei:
            call()
        assert ei.value.code == -4
    f.check_state()                                  # still a valid pseudoflow
    f.close()
    # the same state, repaired by DYN_PR with a generous cap, is exact
    f = dmf.DynMaxFlow.from_graph(g, max_iters=1)
    with pytest.raises(dmf.DMFError):
        f.static_solve()
    st = f.export_state()
    f.close()
    f2 = dmf.DynMaxFlow.from_graph(g)
    f2.import_state(st["cap"], st["res"], st["e"])
    with pytest.raises(dmf.DMFError) as ei:
        f2.flow_value()
    assert ei.value.code == -4
    z = np.zeros(0, np.int32)
    f2.apply_batch(z, z, z, algo="pr")
    _verify(f2, g, "repaired after ENOCONV")
    f2.close()


def test_checkpoint_export_import_roundtrip(dmf):
    """dmf_export_state -> dmf_import_state into a fresh handle of the same graph, a
    DYN_PR repair (k = 0) is a fixed point, then both handles follow the same batches."""
    g = W.rmat(13, 16, 1, 7)
    a = dmf.DynMaxFlow.from_graph(g)
    a.static_solve()
    st = W.CapState(g)
    b0 = W.rmat_batch(g, st, 0.01, 500)
    st.apply(b0)
    a.apply_batch(b0.u, b0.v, b0.new_cap, algo="pp")
    snap = a.export_state()
    b = dmf.DynMaxFlow.from_graph(g)
    b.import_state(snap["cap"], snap["res"], snap["e"])
    z = np.zeros(0, np.int32)
    assert b.apply_batch(z, z, z, algo="pr") == a.flow_value()
    assert np.array_equal(b.min_cut_source_side(), a.min_cut_source_side())
    for j in range(2):
        bb = W.rmat_batch(g, st, 0.01, 501 + j)
        st.apply(bb)
        a.apply_batch(bb.u, bb.v, bb.new_cap, algo="pp")
        b.apply_batch(bb.u, bb.v, bb.new_cap, algo="pp")
        _verify(a, st.graph(), f"a b{j}", check=False)
        _verify(b, st.graph(), f"b b{j}")
    # a corrupted state is rejected and the handle keeps its own state
    F = b.flow_value()
    bad = snap["res"].copy()
    bad[0] += 1
    with pytest.raises(dmf.DMFError) as ei:
        b.import_state(snap["cap"], bad, snap["e"])
    assert ei.value.code == -1
    assert b.flow_value() == F
    b.check_state()
    a.close()
    b.close()


def test_check_level_one(dmf):
    """check_level = 1 runs the device invariant check after every call."""
    g = W.rmat(12, 16, 2, 7)
    f = dmf.DynMaxFlow.from_graph(g, check_level=1)
    f.static_solve()
    st = W.CapState(g)
    for j in range(3):
        b = W.rmat_batch(g, st, 0.02, 600 + j)
        st.apply(b)
        f.apply_batch(b.u, b.v, b.new_cap, algo="pp" if j % 2 == 0 else "pr")
        _verify(f, st.graph(), f"check b{j}", check=False)
    f.close()


def test_device_buffers_on_the_default_stream(dmf):
    """Batches and the mask as CUDA tensors produced by torch kernels on torch's default
    stream, with no host synchronisation in between: the library must be ordered after
    them (cudaStreamLegacy) -- ADVICE r1."""
    import torch
    g = W.rmat(12, 8, 4, 5)
    f = dmf.DynMaxFlow.from_graph(g)
    f.static_solve()
    st = W.CapState(g)
    for j in range(3):
        b = W.rmat_batch(g, st, 0.05, 9 + j)
        st.apply(b)
        # device tensors written by torch kernels (not plain copies) right before the call
        tu = (torch.from_numpy(b.u).cuda() + 0).contiguous()
        tv = (torch.from_numpy(b.v).cuda() * 1).contiguous()
        tc = torch.from_numpy(b.new_cap).cuda().clone()
        mask = torch.full((g.n,), 7, dtype=torch.uint8, device="cuda")
        f.apply_batch(tu, tv, tc, algo="pp")
        f.min_cut_source_side(mask)
        Fo, smin, _ = _oracle(st.graph())
        assert f.flow_value() == Fo
        assert np.array_equal(mask.cpu().numpy(), smin)
    f.close()


def test_certificate_both_outcomes(dmf):
    """DYN_PP warm start: the k_reach certificate holds on small batches (the PP launch
    ends there) and fails when a tiny work budget leaves excess after the warm iteration
    (the MODE_PP_CONT launch runs the full Alg.8 stage 1; later calls then skip the
    certificate for a back-off period); every outcome is exact."""
    g = W.rmat(15, 16, 1, 7)
    for knobs, want in ((dict(), 1), (dict(schedule="async", budget_mul=-1000000, tail_items=1), 0)):
        f = dmf.DynMaxFlow.from_graph(g, **knobs)
        f.static_solve()
        st = W.CapState(g)
        seen = set()
        for j, frac in enumerate([0.001, 0.01, 0.001, 0.01, 0.001, 0.001]):
            b = W.rmat_batch(g, st, frac, 700 + j)
            st.apply(b)
            f.apply_batch(b.u, b.v, b.new_cap, algo="pp")
            if j > 0:                                   # (batch 0 starts from the static labels)
                seen.add(f.stats()["certified"])
            # F and S_min only: the S_max query (MAXCUT launch) would end the warm start
            Fo, smin_o, _ = _oracle(st.graph())
            assert f.flow_value() == Fo, f"cert {knobs} b{j}: F"
            assert np.array_equal(f.min_cut_source_side(), smin_o), f"cert {knobs} b{j}: S_min"
        assert want in seen, f"{knobs}: certificate outcomes {seen}"
        f.close()
