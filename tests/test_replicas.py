"""Replica bookkeeping of the multi-GPU layer, exercised on CPU with gloo and world
size 2 (the GPU path itself is single-GPU per rank and covered by -m gpu)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_05895_b200.replicas import reduce_job, snapshots_for_rank, whole_job_throughput


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    units = [100.0, 250.0][rank]
    ms = [4.0, 5.0][rank]
    r = reduce_job(units, ms, extra_units=units / 2, extra_ms=ms * 2)
    out[rank] = r
    dist.destroy_process_group()


def test_snapshot_assignment():
    assert snapshots_for_rank(8, 0, 1) == list(range(8))
    assert snapshots_for_rank(8, 1, 2) == [1, 3, 5, 7]
    assert sorted(sum((snapshots_for_rank(8, r, 4) for r in range(4)), [])) == list(range(8))


def test_reduce_identity_single_process():
    assert reduce_job(10, 2.0, 3, 4.0) == (10.0, 2.0, 3.0, 4.0)
    assert whole_job_throughput(1000, 2.0) == 500000.0


def test_reduce_gloo_world2():
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    for r in range(2):
        u, ms, eu, ems = out[r]
        assert u == 350.0 and ms == 5.0 and eu == 175.0 and ems == 10.0


def test_bench_launcher_spawns_ranks_gloo():
    """`bench.py --gpus 2` without a launcher re-executes itself under
    torch.distributed.run with 2 ranks; --stub runs the rank bookkeeping on CPU (gloo):
    4 snapshots -> rank 0 takes {0, 2}, rank 1 {1, 3}; whole-job units = SUM, time = MAX."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--snapshots", "4", "--stub"],
                         capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["snapshots_rank0"] == [0, 2]
    assert line["units_all"] == 1000 + 2000 + 3000 + 4000          # every snapshot counted once
    assert line["ms_max"] == max(10 + 30, 20 + 40)                   # slowest rank
    assert abs(line["value"] - 10000 / 0.060) < 1e-6
