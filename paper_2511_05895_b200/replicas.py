"""Multi-GPU layer: independent replicas only.

One push-relabel instance does not shard, so N GPUs run N independent graph
snapshots (one process per GPU, torchrun).  The only collective is one all_reduce
of a few counters outside the timed loop: SUM of work units, MAX of the
device-timed elapsed time (the whole-job time is the slowest rank's)."""
from __future__ import annotations

import torch
import torch.distributed as dist


def env_rank_world():
    import os
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def snapshots_for_rank(num_snapshots: int, rank: int, world: int):
    """Snapshot i goes to rank i mod world."""
    return [i for i in range(num_snapshots) if i % world == rank]


def reduce_job(units: float, elapsed_ms: float, extra_units: float = 0.0, extra_ms: float = 0.0, device=None):
    """All-reduce (SUM units, MAX time) over the default process group; identity at
    world size 1.  Returns (units_all, ms_max, extra_units_all, extra_ms_max)."""
    tot = torch.tensor([float(units), float(extra_units)], dtype=torch.float64, device=device)
    mx = torch.tensor([float(elapsed_ms), float(extra_ms)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    a, b = tot.tolist()
    c, e = mx.tolist()
    return a, c, b, e


def whole_job_throughput(units_all: float, ms_max: float) -> float:
    """Units all ranks processed / the slowest rank's time (weak scaling)."""
    return units_all / (ms_max * 1e-3)
