"""CPU: scene-parallel batch plumbing over torch.distributed (gloo, world size 2)."""

import os
import socket

import numpy as np
import pytest

from paper_2403_19272_b200.batch import gather_metrics, scene_shard


def test_scene_shard_partitions():
    for n in (1, 7, 64):
        for w in (1, 2, 3, 8):
            got = [list(scene_shard(n, w, r)) for r in range(w)]
            flat = [i for g in got for i in g]
            assert flat == list(range(n))
            sizes = [len(g) for g in got]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = {sid: [float(sid), float(rank)] for sid in scene_shard(5, world, rank)}
    merged = gather_metrics(mine, world)
    # max-over-ranks timing reduction used by bench.py
    import torch

    t = torch.tensor([1.0 + rank], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    q.put((rank, merged, float(t)))
    dist.destroy_process_group()


def test_gather_metrics_gloo_world2():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    for rank, merged, tmax in res:
        assert sorted(merged) == [0, 1, 2, 3, 4]
        assert merged[0][1] == 0.0 and merged[4][1] == 1.0
        assert tmax == 2.0
