"""Parallel oracle recomputes over a cumulative batch sequence -- TEST / BENCH
INFRASTRUCTURE ONLY (same import rule as the rest of oracle/).

The dynamic path is checked by a FULL recompute after every batch (SURVEY §8(c)
"Dynamic path: full recompute after every batch").  Every capacity snapshot is a
deterministic function of (workload spec, batch index), so recomputes are
independent: each worker process rebuilds the graph and the batch sequence from
their seeds (workloads/, no method arithmetic), walks the cumulative capacities
forward and runs the single-threaded C oracle at each batch index of its chunk.

    results = recompute(spec, indices, workers=P, deadline_s=..., algo="fifo_pr")

`spec` is a picklable dict understood by workloads.sequence(spec) (graph + batches).
Each result: dict(j, F, smin (uint8[n]) or None, seconds).  With a deadline, a
worker stops starting new solves once it has passed; missing indices are absent.
"""
from __future__ import annotations

import multiprocessing as mp
import os
import time


def _worker(args):
    spec, idxs, algo, want_smin, deadline = args
    import numpy as np  # noqa: F401
    import workloads as W
    import oracle as O
    g, batches = W.sequence(spec)
    st = W.CapState(g)
    out = []
    todo = sorted(idxs)
    j = -1
    for target in todo:
        if deadline is not None and time.time() > deadline:
            break
        while j < target:
            j += 1
            if j >= 0:
                st.apply(batches[j])
        gg = st.graph() if target >= 0 else g
        t0 = time.perf_counter()
        r = O.maxflow(gg, algo)
        dt = time.perf_counter() - t0
        out.append(dict(j=target, F=r["F"], smin=r["smin"] if want_smin else None, seconds=dt))
    return out


def default_workers(mem_per_worker_gb: float = 5.0, cap: int = 8) -> int:
    """min(nproc, cap, available memory / mem_per_worker_gb), at least 1."""
    n = os.cpu_count() or 1
    try:
        avail = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE") / 2 ** 30
        n = min(n, max(1, int(avail // mem_per_worker_gb)))
    except (ValueError, OSError):
        pass
    return max(1, min(n, cap))


def recompute(spec: dict, indices, workers: int | None = None, deadline_s: float | None = None,
              algo: str = "fifo_pr", want_smin: bool = True):
    """Oracle result after each batch index in `indices` (-1 = the initial graph),
    computed on `workers` processes, each taking a contiguous chunk of indices."""
    idx = sorted(set(int(i) for i in indices))
    if not idx:
        return []
    P = max(1, min(workers or default_workers(), len(idx)))
    chunks = [idx[k * len(idx) // P:(k + 1) * len(idx) // P] for k in range(P)]
    deadline = None if deadline_s is None else time.time() + deadline_s
    args = [(spec, c, algo, want_smin, deadline) for c in chunks if c]
    if len(args) == 1:
        res = [_worker(args[0])]
    else:
        ctx = mp.get_context("spawn")
        with ctx.Pool(len(args)) as pool:
            res = pool.map(_worker, args)
    out = [r for part in res for r in part]
    out.sort(key=lambda r: r["j"])
    return out


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"
