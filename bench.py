#!/usr/bin/env python
"""bench.py -- dynamic max-flow batch-update throughput on B200 (arXiv 2511.05895).

Workload (BASELINE.json configs[1]): RMAT-20 (2^20 vertices,
16.09M merged edges, caps U[1,1000]), static solve, then cumulative mixed batches
of 1% of the edges (k = 160,869) biased x10 toward s-out / t-in edges.

A STEP = one pass of the hot path over one batch: dmf_apply_batch (validation,
Updates Processing, Dynamic Push-Pull repair to convergence, flow value) followed
by dmf_min_cut_source_side (S_min mask).  `value` = edge updates per second over
the timed steps with the batches already resident in HBM; `e2e` = the same with
the batch in pinned host memory (H2D inside the timed region) and F + the S_min
mask read back to the host every step.

N > 1 (torchrun): every rank runs an independent RMAT-20 replica (graph seed
1 + rank) -- "replicas only"; one NCCL all_reduce of the counters
and a MAX over ranks of the device-timed elapsed time, outside the timed loop.

--impl reference: the CPU oracle (oracle/, plain C, single thread) timed per step
on the same workload: apply the batch to the capacity table + full recompute.
"""
from __future__ import annotations

import argparse
import json
import os
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

# Algorithmic bytes per unit of work.
B_BFS_VERTEX = 12      # row_ptr pair (8) + height write (4)
B_BFS_SLOT = 8         # dst (4) + mirror/forward residual (4)
B_DIS_VERTEX = 20      # row_ptr (8) + e (8) + height (4)
B_DIS_SLOT = 12        # dst (4) + residual (4) + neighbour height (4)
B_PUSH = 24            # rev (4) + 4 residual atomics... counted as 2 res + 2 e (SURVEY: ~24 B)
B_RIE_SLOT = 12
B_BATCH_ENTRY = 60     # 12 B input + lookup + cap/res/rres r/w + 2 e atomics
B_RESET_VERTEX = 12    # e read (8) + height write (4)


def algorithmic_bytes(st: dict, n: int) -> int:
    """Bytes the method itself must move in one launch (SURVEY §8(d) unit costs x the
    launch's own work counters); + 9 B/vertex for the final F reduction / part pass."""
    return int(st["bfs_vertices"] * B_BFS_VERTEX + st["bfs_slots"] * B_BFS_SLOT
               + st["discharge_vertices"] * B_DIS_VERTEX + st["discharge_slots"] * B_DIS_SLOT
               + st["pushes"] * B_PUSH + st["rie_slots"] * B_RIE_SLOT
               + st["batch_entries"] * B_BATCH_ENTRY + st["reset_vertices"] * B_RESET_VERTEX + n * 9)


def phase_roofline(per: list, peak: float) -> dict:
    """Per-step achieved algorithmic GB/s of the three method steps the north star names,
    from the in-kernel phase clock (one persistent kernel: ncu cannot split its phases):
    global relabel (BFS levels + RESET), discharge (+ RIE), batch update (prologue).
    Medians over the timed steps; frac against the same measured HBM peak."""
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


def make_workload(rank: int, frac: float, nb: int, seed_base: int = 100, scale: int = 20):
    """RMAT-`scale` snapshot of this rank (graph seed 1 + rank) and its cumulative batches:
    scale 20 = BASELINE config 2 (the default bench line), 22 = one config-5 snapshot."""
    g = W.rmat(scale, 16, 1 + rank, 7)
    st = W.CapState(g)
    batches = []
    for j in range(nb):
        b = W.rmat_batch(g, st, frac, seed_base + j)
        st.apply(b)
        batches.append(b)
    return g, batches


def cpu_oracle_sample(g, b, algo="fifo_pr"):
    """Time one full oracle recompute after one batch (bounded sample)."""
    import oracle as O
    st = W.CapState(g)
    st.apply(b)
    gg = st.graph()
    t0 = time.perf_counter()
    r = O.maxflow(gg, algo)
    dt = time.perf_counter() - t0
    return dt, r["F"]


def run_reference(args):
    """--impl reference: the CPU oracle on the same workload (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle as O
    O.build()
    nb = args.warmup + args.steps
    g, batches = make_workload(0, args.frac, nb, scale=20 if args.workload == "rmat20" else 22)
    st = W.CapState(g)
    times, k_tot = [], 0
    for j, b in enumerate(batches):
        st.apply(b)
        gg = st.graph()
        t0 = time.perf_counter()
        O.maxflow(gg, args.oracle_algo)
        dt = time.perf_counter() - t0
        if j >= args.warmup:
            times.append(dt)
            k_tot += b.k
    total = sum(times)
    value = k_tot / total
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic", "config": config_dict(g, args, batches[0].k),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"{len(times)} steps: batch applied to the capacity table + full "
                                       f"{args.oracle_algo} recompute of RMAT-20 (single thread)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def config_dict(g, args, k):
    wl = ("config2 RMAT-20 (2^20 V, ef 16, caps U[1,1000]) + cumulative 1% mixed batches" if args.workload == "rmat20"
          else "config5 RMAT-22 snapshot per rank (2^22 V, ef 16, caps U[1,1000], graph seed 1 + rank) "
               "+ cumulative 1% mixed batches")
    return {"workload": wl,
            "n": int(g.n), "m": int(g.m), "batch_k": int(k), "batch_frac": args.frac, "algo": args.algo,
            "step": "dmf_apply_batch + dmf_min_cut_source_side" if not args.no_cut else "dmf_apply_batch",
            "l2": "inputs larger than L2 (slot arrays 28 B/slot x S slots: 0.88 GB (RMAT-20) / 3.6 GB (RMAT-22) >> 126 MB L2)",
            "parallelism": f"replicas x{args.gpus}"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="dmf", choices=["dmf", "reference"])
    ap.add_argument("--algo", default="pp", choices=["pp", "pr"])
    ap.add_argument("--workload", default="rmat20", choices=["rmat20", "rmat22"],
                    help="rmat20 = BASELINE config 2 (default); rmat22 = config 5 (one RMAT-22 snapshot per rank)")
    ap.add_argument("--frac", type=float, default=0.01)
    ap.add_argument("--no-cut", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--oracle-algo", default="fifo_pr")
    ap.add_argument("--static-reps", type=int, default=3)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    import paper_2511_05895_b200 as P
    from paper_2511_05895_b200.replicas import reduce_job

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)

    K, Wm = args.steps, args.warmup
    nb = Wm + 2 * K                       # warm-up, device-resident timed steps, e2e timed steps
    g, batches = make_workload(rank, args.frac, nb, scale=20 if args.workload == "rmat20" else 22)
    f = P.DynMaxFlow.from_graph(g, algo=args.algo)
    stream = f.stream

    # ---- static solve (the baseline a dynamic repair is compared with)
    f.static_solve()
    F_static0 = f.flow_value()
    st_static = f.stats()

    # batches resident in HBM
    dbat = [(torch.from_numpy(b.u).to(dev), torch.from_numpy(b.v).to(dev), torch.from_numpy(b.new_cap).to(dev))
            for b in batches]
    hbat = [(torch.from_numpy(b.u).pin_memory(), torch.from_numpy(b.v).pin_memory(),
             torch.from_numpy(b.new_cap).pin_memory()) for b in batches]
    dmask = torch.empty(g.n, dtype=torch.uint8, device=dev)
    hmask = torch.empty(g.n, dtype=torch.uint8).pin_memory()
    torch.cuda.synchronize()

    raw = [P.Stats() for _ in range(nb)]

    def step(j, host=False):
        u, v, c = (hbat if host else dbat)[j]
        f.apply_batch(u, v, c, algo=args.algo)
        f.raw_stats(raw[j])                      # ctypes copy only; dicts are built after timing
        if not args.no_cut:
            f.min_cut_source_side(hmask if host else dmask)

    for j in range(Wm):
        step(j)

    clk = ClockSampler(dev.index if dev.index is not None else 0)
    clk.start()
    time.sleep(0.2)
    # ---- timed: device-resident batches
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = f.stats()["kernel_launches"]
    e0.record(stream)
    k_tot = 0
    for j in range(Wm, Wm + K):
        step(j)
        k_tot += batches[j].k
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    elapsed_ms = e0.elapsed_time(e1)
    launches = f.stats()["kernel_launches"] - launches0
    per = [P.DynMaxFlow.stats_to_dict(raw[j]) for j in range(Wm, Wm + K)]
    kernel_ms = [p_["device_ms"] for p_ in per]
    alg_bytes = [algorithmic_bytes(p_, g.n) for p_ in per]

    # ---- timed: end to end from pinned host buffers, F + mask back to the host
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    k_e2e = 0
    for j in range(Wm + K, Wm + 2 * K):
        step(j, host=True)
        k_e2e += batches[j].k
    torch.cuda.synchronize()
    e2e_ms = 1e3 * (time.perf_counter() - t0)
    if world > 1:
        dist.barrier()
    clocks = clk.stop()

    # ---- static re-solve on the final capacities (speedup baseline) + parity of F
    F_dyn = f.flow_value()
    mask_dyn = f.min_cut_source_side() if not args.no_cut else None
    # both static solves this build has: Alg.1 and the static push-pull variant
    # (P:515-518); the speedup is taken against the FASTER one
    static_ms, static_pp_ms = [], []
    for _ in range(args.static_reps):
        f.static_solve()
        static_ms.append(f.stats()["device_ms"])
        assert f.flow_value() == F_dyn, f"static re-solve F={f.flow_value()} != dynamic F={F_dyn}"
        f.static_solve_pp()
        static_pp_ms.append(f.stats()["device_ms"])
        assert f.flow_value() == F_dyn, f"static push-pull F={f.flow_value()} != dynamic F={F_dyn}"
    if mask_dyn is not None:
        assert np.array_equal(f.min_cut_source_side(), mask_dyn)

    # ---- reduce over ranks (one NCCL all_reduce each, outside the timed loops)
    k_all, el_max, k_e2e_all, e2e_max = reduce_job(k_tot, elapsed_ms, k_e2e, e2e_ms, device=dev)

    if rank == 0:
        peak, peak_src = peaks()
        km = float(np.mean(kernel_ms))
        ab = float(np.mean(alg_bytes))
        achieved = ab / (km * 1e-3) / 1e9
        traffic = None
        tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tp):
            try:
                traffic = json.load(open(tp)).get("k_solve_pp_bytes_per_launch")
            except Exception:
                traffic = None
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            dt, Fo = cpu_oracle_sample(g, batches[0], args.oracle_algo)
            cpu = {"value": batches[0].k / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
                   "sample": f"one full {args.oracle_algo} recompute of {args.workload.upper()} after batch 0 "
                             f"(k={batches[0].k}), single thread, {dt:.2f} s"}
        ms_step = el_max / K
        static_alg1 = float(np.median(static_ms))
        static_pp = float(np.median(static_pp_ms))
        static_med = min(static_alg1, static_pp)
        apply_ms = float(np.median([p["device_ms"] for p in per]))
        med = lambda key: float(np.median([p[key] for p in per]))  # noqa: E731
        line = {
            "metric": METRIC, "value": k_all / (el_max * 1e-3), "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": Wm, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": config_dict(g, args, batches[0].k),
            "e2e": {"value": k_e2e_all / (e2e_max * 1e-3), "unit": UNIT,
                    "h2d_bytes_per_step": int(3 * 4 * batches[0].k),
                    "d2h_bytes_per_step": int(8 + (0 if args.no_cut else g.n))},
            "gpu_launches": int(launches),
            "phase_roofline": phase_roofline(per, peak),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": f"k_solve (mode {args.algo.upper()} batch launch)",
                         "algorithmic_bytes_per_launch": ab, "kernel_ms": km, "peak_source": peak_src},
            "cpu_baseline": cpu,
            "clocks": {k: clocks[k] for k in ("sm_mhz", "sm_max_mhz", "reasons")},
            "batch_apply_ms_median": apply_ms,
            # device time of the e2e steps' own launches (later cumulative batches): separates the
            # host-path overhead (copies, syncs) from the batches being different
            "e2e_batch_device_ms_median": float(np.median([P.DynMaxFlow.stats_to_dict(raw[j])["device_ms"]
                                                           for j in range(Wm + K, Wm + 2 * K)])),
            "static_solve_ms_median": static_med,
            "static_solve_ms_median_by_variant": {"alg1": static_alg1, "static_push_pull": static_pp},
            "speedup_vs_static": static_med / apply_ms,
            "edges_per_s": g.m / (apply_ms * 1e-3),
            "static_edges_per_s": g.m / (static_med * 1e-3),
            "flow": {"F_static_initial": F_static0, "F_final": F_dyn},
            "phase_us_median": {k: med(k) for k in ("t_prologue_us", "t_reset_us", "t_bfs_us", "t_discharge_us",
                                                     "t_rie_us", "t_epilogue_us")},
            "per_batch_median": {k: med(k) for k in ("iterations", "rounds", "bfs_levels", "bfs_slots",
                                                     "discharge_vertices", "activations", "pushes", "relabels",
                                                     "stage2_vertices")},
            "static_solve_stats": {k: st_static[k] for k in ("iterations", "rounds", "bfs_levels", "bfs_slots",
                                                             "discharge_slots", "pushes", "relabels",
                                                             "device_ms")},
        }
        print(json.dumps(line))
    f.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
