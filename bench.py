#!/usr/bin/env python
"""bench.py -- dynamic max-flow batch-update throughput on B200 (arXiv 2511.05895).

Workload (default): ONE config-5 snapshot, the largest RMAT graph of BASELINE.json
(RMAT-22: 2^22 vertices, 65.2M merged edges, caps U[1,1000]; the north-star target
"at least 10x faster than the static re-solve" is stated on it), static solve, then
cumulative mixed batches of 1% of the edges (k = 652,450) biased x10 toward s-out /
t-in edges.  `--workload rmat20` runs config 2 (RMAT-20) instead; the default run
also reports the RMAT-20 figures under "rmat20".

A STEP = one pass of the hot path over one batch: dmf_apply_batch (validation,
Updates Processing, Dynamic Push-Pull repair to convergence, flow value) plus
dmf_min_cut_source_side (S_min mask).
  * value  -- edge updates / s over the K timed steps, batches already in HBM, device
              time (CUDA events on the handle's stream).
  * e2e    -- the SAME K batches on a second handle through the public API from pinned
              host buffers (H2D inside the call) with F and the S_min mask read back to
              the host every step; host wall clock with a device sync.
  * speedup_vs_static -- for EVERY timed batch j a third handle solves the capacity
              snapshot after batch j from scratch (dmf_static_solve and
              dmf_static_solve_pp, the faster counts); median over j of static / batch.
N > 1: `python bench.py --gpus N` re-executes itself under torch.distributed.run
(N ranks, one per GPU); rank r takes the snapshots i = r mod N of `--snapshots`
(default N: one snapshot per rank, graph seed 1 + i, weak scaling).  Replicas only
(DESIGN.md §7): no data-path collective; one NCCL all_reduce of the counters and a
MAX of the device-timed elapsed time, outside the timed loop.

--impl reference: the CPU oracle (oracle/, plain C, single thread per solve) on the
same workload: a full recompute per batch on a pool of worker processes.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

METRIC = "dynamic batch update ms and speedup vs static GPU re-solve; edges/s, HBM GB/s"
UNIT = "edge updates/s"
DEFAULT_STEPS, DEFAULT_WARMUP = 20, 5

# Algorithmic bytes per unit of work.
B_BFS_VERTEX = 12      # row_ptr pair (8) + height write (4)
B_BFS_SLOT = 8         # dst (4) + mirror/forward residual (4)
B_DIS_VERTEX = 20      # row_ptr (8) + e (8) + height (4)
B_DIS_SLOT = 12        # dst (4) + residual (4) + neighbour height (4)
B_PUSH = 24            # rev (4) + 2 residual + 2 excess updates (SURVEY: ~24 B)
B_RIE_SLOT = 12
B_BATCH_ENTRY = 60     # 12 B input + lookup + cap/res/rres r/w + 2 e atomics
B_RESET_VERTEX = 12    # e read (8) + height write (4)


def workload_spec(workload: str, warmup: int, steps: int, snapshot: int = 0, frac: float = 0.01) -> dict:
    """The batch sequence one bench replica runs: warm-up batches, then the timed ones."""
    scale = {"rmat22": 22, "rmat20": 20}[workload]
    return dict(kind="rmat", scale=scale, edge_factor=16, seed_graph=1 + snapshot, seed_caps=7, frac=frac,
                nb=warmup + steps, seed_base=100)


def algorithmic_bytes(st: dict, n: int) -> int:
    """Bytes the method itself must move in one launch (SURVEY §8(d) unit costs x the
    launch's own work counters); + 9 B/vertex for the final F reduction / part pass."""
    return int(st["bfs_vertices"] * B_BFS_VERTEX + st["bfs_slots"] * B_BFS_SLOT
               + st["discharge_vertices"] * B_DIS_VERTEX + st["discharge_slots"] * B_DIS_SLOT
               + st["pushes"] * B_PUSH + st["rie_slots"] * B_RIE_SLOT
               + st["batch_entries"] * B_BATCH_ENTRY + st["reset_vertices"] * B_RESET_VERTEX + n * 9)


def cut_algorithmic_bytes(bfs_v: int, bfs_slots: int, n: int) -> int:
    """Bytes of one S_min query (k_reach<false>): root sweep (e read + label write, 12 B
    per vertex), BFS (12 B per labelled vertex, 8 B per scanned slot), mask sweep (label
    read + mask write, 5 B per vertex)."""
    return int(n * 12 + bfs_v * B_BFS_VERTEX + bfs_slots * B_BFS_SLOT + n * 5)


def phase_roofline(per: list, peak: float) -> dict:
    """Per-step achieved algorithmic GB/s of the three method steps the north star names,
    from the in-kernel phase clock (one persistent kernel: ncu cannot split its phases):
    global relabel (BFS levels + RESET), discharge (+ RIE), batch update (prologue)."""
    def row(bytes_fn, us_keys):
        vals = []
        for p_ in per:
            us = sum(p_[k] for k in us_keys)
            if us > 0:
                vals.append(bytes_fn(p_) / (us * 1e-6) / 1e9)
        a = float(np.median(vals)) if vals else 0.0
        return {"achieved_gbs": a, "frac": a / peak if peak else None,
                "us_median": float(np.median([sum(p_[k] for k in us_keys) for p_ in per]))}
    return {
        "global_relabel": row(lambda p_: p_["bfs_vertices"] * B_BFS_VERTEX + p_["bfs_slots"] * B_BFS_SLOT
                              + p_["reset_vertices"] * B_RESET_VERTEX, ("t_bfs_us", "t_reset_us")),
        "discharge": row(lambda p_: p_["discharge_vertices"] * B_DIS_VERTEX + p_["discharge_slots"] * B_DIS_SLOT
                         + p_["pushes"] * B_PUSH + p_["rie_slots"] * B_RIE_SLOT, ("t_discharge_us", "t_rie_us")),
        "batch_update": row(lambda p_: p_["batch_entries"] * B_BATCH_ENTRY, ("t_prologue_us",)),
        "note": "phase clock = block 0's barrier-to-barrier laps; bytes = SURVEY 8(d) unit costs x the phase's counters",
    }


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, val in zip(names, parts[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def pctl(x, q):
    return float(np.percentile(np.asarray(x, np.float64), q)) if len(x) else None


_T0 = time.time()


def progress(msg: str) -> None:
    """Stage marks on stderr (the JSON line stays the only stdout output)."""
    print(f"[bench {time.time() - _T0:7.1f}s] {msg}", file=sys.stderr, flush=True)


def run_snapshot(P, torch, dev, spec, W_, K, algo, no_cut=False):
    """One replica: handles A (device-resident timed steps), B (e2e from host buffers on
    the same batches) and C (static re-solves of the same capacity snapshots)."""
    g, batches = W.sequence(spec)
    out = {"n": g.n, "m": g.m, "k": batches[0].k}
    dbat = [(torch.from_numpy(b.u).to(dev), torch.from_numpy(b.v).to(dev), torch.from_numpy(b.new_cap).to(dev))
            for b in batches]
    hbat = [(torch.from_numpy(b.u).pin_memory(), torch.from_numpy(b.v).pin_memory(),
             torch.from_numpy(b.new_cap).pin_memory()) for b in batches]
    dmask = torch.empty(g.n, dtype=torch.uint8, device=dev)
    hmask = torch.empty(g.n, dtype=torch.uint8).pin_memory()
    torch.cuda.synchronize()

    progress(f"snapshot {spec.get('scale')} built (n={g.n}); A: device-resident")
    # ---- A: device-resident
    fa = P.DynMaxFlow.from_graph(g, algo=algo)
    fa.static_solve()
    out["F_static_initial"] = fa.flow_value()
    raw = [P.Stats() for _ in batches]
    qms, qalg = [], []
    for j in range(W_):
        u, v, c = dbat[j]
        fa.apply_batch(u, v, c, algo=algo)
        if not no_cut:
            fa.min_cut_source_side(dmask)
    stream = fa.stream
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
    launches0 = fa.stats()["kernel_launches"]
    ev[0].record(stream)
    for i, j in enumerate(range(W_, W_ + K)):
        u, v, c = dbat[j]
        fa.apply_batch(u, v, c, algo=algo)
        fa.raw_stats(raw[j])
        if not no_cut:
            fa.min_cut_source_side(dmask)
            rq = fa.raw_stats()
            qms.append(rq.query_ms)
            qalg.append(cut_algorithmic_bytes(rq.query_bfs_vertices, rq.query_bfs_slots, g.n))
        ev[i + 1].record(stream)
    torch.cuda.synchronize()
    out["elapsed_ms"] = ev[0].elapsed_time(ev[K])
    out["step_ms"] = [ev[i].elapsed_time(ev[i + 1]) for i in range(K)]
    out["launches"] = fa.stats()["kernel_launches"] - launches0
    out["per"] = [P.DynMaxFlow.stats_to_dict(raw[j]) for j in range(W_, W_ + K)]
    out["query_ms"] = qms
    out["query_alg_bytes"] = qalg
    out["F_final"] = fa.flow_value()
    out["k_timed"] = int(sum(batches[j].k for j in range(W_, W_ + K)))
    fa.close()

    progress("B: end to end")
    # ---- B: end to end through the public API, same batches, pinned host buffers
    fb = P.DynMaxFlow.from_graph(g, algo=algo)
    fb.static_solve()
    for j in range(W_):
        u, v, c = hbat[j]
        fb.apply_batch(u, v, c, algo=algo)
        if not no_cut:
            fb.min_cut_source_side(hmask)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e2e_steps = []
    for j in range(W_, W_ + K):
        ts = time.perf_counter()
        u, v, c = hbat[j]
        fb.apply_batch(u, v, c, algo=algo)       # H2D of the batch inside the call; returns F on the host
        if not no_cut:
            fb.min_cut_source_side(hmask)        # D2H of the S_min mask
        e2e_steps.append(1e3 * (time.perf_counter() - ts))
    torch.cuda.synchronize()
    out["e2e_ms"] = 1e3 * (time.perf_counter() - t0)
    out["e2e_step_ms"] = e2e_steps
    assert fb.flow_value() == out["F_final"], "e2e handle diverged from the device-resident one"
    fb.close()

    progress("C: static re-solves")
    # ---- C: static re-solve of every timed capacity snapshot (the paper's baseline)
    fc = P.DynMaxFlow.from_graph(g, algo=algo)
    fc.static_solve()
    st_alg1, st_pp, st_cut = [], [], []
    for j in range(W_ + K):
        u, v, c = dbat[j]
        fc.apply_batch(u, v, c, algo="pp")
        if j < W_:
            continue
        Fd = fc.flow_value()
        fc.static_solve()
        st_alg1.append(fc.stats()["device_ms"])
        assert fc.flow_value() == Fd
        fc.static_solve_pp()
        st_pp.append(fc.stats()["device_ms"])
        assert fc.flow_value() == Fd
        if not no_cut:
            fc.min_cut_source_side(dmask)              # S_min of the static solution (MINCUT launch)
            st_cut.append(fc.raw_stats().query_ms)
    out["static_stats"] = fc.stats()
    fc.close()
    out["static_alg1_ms"] = st_alg1
    out["static_pp_ms"] = st_pp
    out["static_cut_ms"] = st_cut
    return out


def summarize(snaps, K, peak):
    per = [p for s in snaps for p in s["per"]]
    batch_ms = [p["device_ms"] for p in per]
    static_ms = [min(a, b) for s in snaps for a, b in zip(s["static_alg1_ms"], s["static_pp_ms"])]
    ratio = [st / p["device_ms"] for s in snaps for st, p in
             zip([min(a, b) for a, b in zip(s["static_alg1_ms"], s["static_pp_ms"])], s["per"])]
    n = snaps[0]["n"]
    alg = [algorithmic_bytes(p, n) for p in per]
    km = float(np.mean(batch_ms))
    ab = float(np.mean(alg))
    med = lambda key: float(np.median([p[key] for p in per]))  # noqa: E731
    qms = [x for s in snaps for x in s["query_ms"]]
    scut = [x for s in snaps for x in s["static_cut_ms"]]
    with_cut = None
    if qms and scut:
        with_cut = (float(np.median(static_ms)) + float(np.median(scut))) / \
                   (float(np.median(batch_ms)) + float(np.median(qms)))
    qab = [x for s in snaps for x in s.get("query_alg_bytes", [])]
    cut_roof = None
    if qms and qab:
        cm = float(np.mean(qms))
        ca = float(np.mean(qab))
        cut_roof = {"kernel": "k_reach<false> (S_min query)", "bound": "hbm", "achieved": ca / (cm * 1e-3) / 1e9,
                    "peak": peak, "unit": "GB/s", "frac": ca / (cm * 1e-3) / 1e9 / peak,
                    "algorithmic_bytes_per_launch": ca, "kernel_ms": cm}
    return {
        "cut_roofline": cut_roof,
        "cut_query_ms": {"p50": pctl(qms, 50), "p90": pctl(qms, 90),
                         "static_p50": pctl(scut, 50)} if qms else None,
        "speedup_vs_static_with_cut": with_cut,
        "batch_ms": {"p50": pctl(batch_ms, 50), "p90": pctl(batch_ms, 90), "mean": km},
        "static_ms": {"p50": pctl(static_ms, 50), "p90": pctl(static_ms, 90),
                      "alg1_p50": pctl([x for s in snaps for x in s["static_alg1_ms"]], 50),
                      "static_push_pull_p50": pctl([x for s in snaps for x in s["static_pp_ms"]], 50)},
        "speedup_vs_static": float(np.median(static_ms)) / float(np.median(batch_ms)),
        "speedup_vs_static_per_batch": {"p50": pctl(ratio, 50), "p10": pctl(ratio, 10)},
        "step_ms": {"p50": pctl([x for s in snaps for x in s["step_ms"]], 50),
                    "p90": pctl([x for s in snaps for x in s["step_ms"]], 90)},
        "e2e_step_ms": {"p50": pctl([x for s in snaps for x in s["e2e_step_ms"]], 50),
                        "p90": pctl([x for s in snaps for x in s["e2e_step_ms"]], 90)},
        "edges_per_s": snaps[0]["m"] / (float(np.median(batch_ms)) * 1e-3),
        "static_edges_per_s": snaps[0]["m"] / (float(np.median(static_ms)) * 1e-3),
        "roofline": {"bound": "hbm", "achieved": ab / (km * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                     "frac": ab / (km * 1e-3) / 1e9 / peak, "algorithmic_bytes_per_launch": ab, "kernel_ms": km},
        "phase_roofline": phase_roofline(per, peak),
        "phase_us_median": {k: med(k) for k in ("t_prologue_us", "t_reset_us", "t_bfs_us", "t_discharge_us",
                                                 "t_rie_us", "t_epilogue_us")},
        "per_batch_median": {k: med(k) for k in ("iterations", "rounds", "bfs_levels", "bfs_slots", "discharge_vertices",
                                                 "discharge_slots", "pushes", "relabels", "stage2_vertices",
                                                 "gap_levels", "gap_skips")},
        "per_launch": [{"alg_bytes": a, "ms": p["device_ms"]} for a, p in zip(alg, per)],
    }


def cpu_baseline(spec, W_, K, k, budget_s):
    """The oracle (as it stands) on the timed batches' capacity snapshots, a pool of
    worker processes, bounded by budget_s of wall time."""
    from oracle.pool import recompute, default_workers, cpu_model
    Pw = default_workers(mem_per_worker_gb=5.0 if spec["scale"] >= 22 else 2.0, cap=os.cpu_count() or 1)
    t0 = time.time()
    res = recompute(spec, list(range(W_, W_ + K)), workers=Pw, deadline_s=budget_s, want_smin=False)
    wall = time.time() - t0
    secs = [r["seconds"] for r in res]
    return {"value": (k * len(res)) / wall if res else None, "unit": UNIT, "cores": Pw, "kind": "oracle",
            "sample": f"{len(res)} of the {K} timed batches: full two-phase FIFO push-relabel recompute of the "
                      f"capacity snapshot after each (plain C, single thread per solve) on a pool of {Pw} worker "
                      f"processes ({cpu_model()}); each worker also rebuilds the graph and its batches; "
                      f"bounded by {budget_s:.0f} s of wall time",
            "per_solve_s_median": float(np.median(secs)) if secs else None, "pool_wall_s": wall,
            "workers": Pw, "cpu_model": cpu_model()}


def run_reference(args):
    """--impl reference: the CPU oracle, as it stands, on the same workload and metric
    (rank 0 only; other ranks exit 0 without work)."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    import oracle as O
    from oracle.pool import recompute, default_workers, cpu_model
    O.build()
    spec = workload_spec(args.workload, args.warmup, args.steps, frac=args.frac)
    g, batches = W.sequence(dict(spec, nb=1))
    k = batches[0].k
    Pw = default_workers(mem_per_worker_gb=5.0 if spec["scale"] >= 22 else 2.0, cap=os.cpu_count() or 1)
    t0 = time.time()
    res = recompute(spec, list(range(args.warmup, args.warmup + args.steps)), workers=Pw,
                    deadline_s=args.cpu_budget_s, want_smin=False)
    wall = time.time() - t0
    value = k * len(res) / wall if res else None
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": len(res), "warmup": args.warmup, "ms_per_step": 1e3 * wall / max(1, len(res)),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic", "config": config_dict(g.n, g.m, args, k),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": Pw, "kind": "oracle",
                             "sample": f"{len(res)} of the {args.steps} timed batches of the GPU arm: full FIFO "
                                       f"push-relabel recompute per batch, {Pw} worker processes ({cpu_model()}), "
                                       f"bounded by {args.cpu_budget_s:.0f} s; per-solve median "
                                       f"{np.median([r['seconds'] for r in res]) if res else float('nan'):.1f} s"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def config_dict(n, m, args, k):
    wl = {"rmat22": "config5 snapshot: RMAT-22 (2^22 V, ef 16, caps U[1,1000], graph seed 1 + snapshot) "
                    "+ cumulative 1% mixed batches (the largest RMAT graph of BASELINE.json)",
          "rmat20": "config2 RMAT-20 (2^20 V, ef 16, caps U[1,1000]) + cumulative 1% mixed batches"}[args.workload]
    return {"workload": wl, "n": int(n), "m": int(m), "batch_k": int(k), "batch_frac": args.frac,
            "algo": args.algo, "snapshots": args.snapshots,
            "step": "dmf_apply_batch + dmf_min_cut_source_side" if not args.no_cut else "dmf_apply_batch",
            "l2": "inputs larger than L2 (slot arrays 28 B/slot x S slots: 3.6 GB (RMAT-22) / 0.88 GB (RMAT-20) "
                  ">> 126 MB L2)",
            "parallelism": f"replicas x{args.gpus} (snapshot i on rank i mod {args.gpus})"}


def run_stub(args):
    """--stub: the multi-rank plumbing of main() on CPU with gloo -- rank / snapshot
    assignment, the SUM / MAX reduction and rank 0's whole-job line -- with a
    deterministic stand-in for the per-snapshot GPU work (tests/test_replicas.py)."""
    import torch.distributed as dist
    from paper_2511_05895_b200.replicas import reduce_job, snapshots_for_rank
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"WORLD_SIZE={world} but --gpus {args.gpus}")
    if world > 1:
        dist.init_process_group("gloo")
    mine = snapshots_for_rank(args.snapshots, rank, world)
    k = [1000 * (1 + i) for i in mine]                 # stand-in work units per snapshot
    ms = [10.0 * (1 + i) for i in mine]                # stand-in device time per snapshot
    k_all, ms_max, _, _ = reduce_job(sum(k), sum(ms), 0, 0)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": k_all / (ms_max * 1e-3), "unit": UNIT, "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup, "scaling": "weak", "stub": True,
                          "snapshots_rank0": mine, "units_all": k_all, "ms_max": ms_max}))
    if world > 1:
        dist.destroy_process_group()


def relaunch_under_torchrun(args):
    """`--gpus N` without a launcher: re-execute under torch.distributed.run, N ranks."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=DEFAULT_STEPS)
    ap.add_argument("--warmup", type=int, default=DEFAULT_WARMUP)
    ap.add_argument("--impl", default="dmf", choices=["dmf", "reference"])
    ap.add_argument("--algo", default="pp", choices=["pp", "pr"])
    ap.add_argument("--workload", default="rmat22", choices=["rmat22", "rmat20"])
    ap.add_argument("--snapshots", type=int, default=0, help="total snapshots over all ranks (0: one per rank)")
    ap.add_argument("--frac", type=float, default=0.01)
    ap.add_argument("--no-cut", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the RMAT-20 figures of the default run")
    ap.add_argument("--cpu-budget-s", type=float, default=150.0)
    ap.add_argument("--stub", action="store_true",
                    help="launcher / replica bookkeeping test on CPU (gloo): no GPU work, a stub per snapshot")
    args = ap.parse_args()
    if args.snapshots <= 0:
        args.snapshots = args.gpus
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        return run_reference(args)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch_under_torchrun(args))
    if args.stub:
        return run_stub(args)

    import torch
    import torch.distributed as dist
    import paper_2511_05895_b200 as P
    from paper_2511_05895_b200.replicas import reduce_job, snapshots_for_rank

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"WORLD_SIZE={world} but --gpus {args.gpus}")
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)
    K, Wm = args.steps, args.warmup

    mine = snapshots_for_rank(args.snapshots, rank, world)
    clk = ClockSampler(dev.index if dev.index is not None else 0)
    clk.start()
    snaps = []
    for i in mine:
        spec = workload_spec(args.workload, Wm, K, snapshot=i, frac=args.frac)
        if world > 1:
            dist.barrier()
        snaps.append(run_snapshot(P, torch, dev, spec, Wm, K, args.algo, args.no_cut))
    clocks = clk.stop()
    k_tot = sum(s["k_timed"] for s in snaps)
    el = sum(s["elapsed_ms"] for s in snaps)
    e2e = sum(s["e2e_ms"] for s in snaps)
    k_all, el_max, k_e2e_all, e2e_max = reduce_job(k_tot, el, k_tot, e2e, device=dev)

    if rank == 0:
        peak, peak_src = peaks()
        summ = summarize(snaps, K, peak)
        g0 = snaps[0]
        extra = None
        if world == 1 and args.workload == "rmat22" and not args.no_extra:
            progress("RMAT-20 figures")
            s20 = run_snapshot(P, torch, dev, workload_spec("rmat20", Wm, K, frac=args.frac), Wm, K, args.algo,
                               args.no_cut)
            sm20 = summarize([s20], K, peak)
            extra = {"workload": "config2 RMAT-20 (2^20 V / 16.1M E), same protocol",
                     "value": s20["k_timed"] / (s20["elapsed_ms"] * 1e-3),
                     "e2e_value": s20["k_timed"] / (s20["e2e_ms"] * 1e-3),
                     "ms_per_step": s20["elapsed_ms"] / K,
                     **{k: sm20[k] for k in ("batch_ms", "static_ms", "speedup_vs_static",
                                               "speedup_vs_static_with_cut", "cut_query_ms", "roofline",
                                               "phase_us_median")}}
        traffic = None
        tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tp):
            try:
                traffic = json.load(open(tp)).get(args.workload, {}).get("dram_bytes_per_launch")
            except Exception:
                traffic = None
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            progress("cpu baseline (oracle pool)")
            cpu = cpu_baseline(workload_spec(args.workload, Wm, K, frac=args.frac), Wm, K, g0["k"], args.cpu_budget_s)
            progress("done")
        roof = summ["roofline"]
        roof.update({"traffic": traffic,
                     "kernel": f"dmf_apply_batch ({args.algo.upper()}): k_solve + k_reach<true> certificate launches",
                     "peak_source": peak_src,
                     "traffic_source": "profiles/ncu_traffic.json: ncu dram__bytes_read+write summed over timed "
                                       "step 0's dmf_apply_batch launches at the recorded commit; their "
                                       "algorithmic bytes are recorded beside it"})
        line = {
            "metric": METRIC, "value": k_all / (el_max * 1e-3), "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": Wm, "ms_per_step": el_max / (K * len(mine)), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": config_dict(g0["n"], g0["m"], args, g0["k"]),
            "e2e": {"value": k_e2e_all / (e2e_max * 1e-3), "unit": UNIT,
                    "h2d_bytes_per_step": int(3 * 4 * g0["k"]),
                    "d2h_bytes_per_step": int(8 + (0 if args.no_cut else g0["n"])),
                    "note": "same batches as value, second handle, host buffers through dmf_apply_batch; "
                            "host wall clock"},
            "gpu_launches": int(sum(s["launches"] for s in snaps)),
            "roofline": roof,
            "cpu_baseline": cpu,
            "clocks": {k: clocks[k] for k in ("sm_mhz", "sm_max_mhz", "reasons")},
            "batch_apply_ms": summ["batch_ms"],
            "static_solve_ms": summ["static_ms"],
            "speedup_vs_static": summ["speedup_vs_static"],
            "speedup_vs_static_with_cut": summ["speedup_vs_static_with_cut"],
            "cut_query_ms": summ["cut_query_ms"], "cut_roofline": summ["cut_roofline"],
            "speedup_vs_static_per_batch": summ["speedup_vs_static_per_batch"],
            "step_ms": summ["step_ms"], "e2e_step_ms": summ["e2e_step_ms"],
            "edges_per_s": summ["edges_per_s"], "static_edges_per_s": summ["static_edges_per_s"],
            "flow": {"F_static_initial": g0["F_static_initial"], "F_final": g0["F_final"]},
            "phase_roofline": summ["phase_roofline"],
            "phase_us_median": summ["phase_us_median"],
            "per_batch_median": summ["per_batch_median"],
            "first_timed_launch": summ["per_launch"][0],
            "rmat20": extra,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
