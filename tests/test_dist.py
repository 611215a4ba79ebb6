"""Data-parallel host logic on CPU (gloo, world_size 2): batch sharding and the
weighted flat-gradient all-reduce equal the reference's global batch mean
(neural.py:472-477) for even and uneven splits."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from paper_2509_24677_b200.train import allreduce_weighted, shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(0)
        per_sample = rng.standard_normal((7, 50))  # identical on every rank
        out = []
        for batch in ([0, 1, 2, 3], [4, 5, 6], [6]):
            mine = shard(batch, rank, world)
            local = torch.tensor(per_sample[mine].mean(0) if mine else np.zeros(50))
            allreduce_weighted(local, len(mine) / len(batch))
            out.append(local.numpy())
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_shard_covers_batch_once():
    from paper_2509_24677_b200.train import shard
    batch = [9, 3, 5, 1, 7]
    parts = [shard(batch, r, 3) for r in range(3)]
    assert sorted(sum(parts, [])) == sorted(batch)
    assert shard([4], 1, 2) == []


def test_weighted_allreduce_equals_global_mean_gloo():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    per_sample = np.random.default_rng(0).standard_normal((7, 50))
    for k, batch in enumerate(([0, 1, 2, 3], [4, 5, 6], [6])):
        want = per_sample[batch].mean(0)
        for r in range(2):
            assert np.allclose(res[r][k], want, atol=1e-12), (r, k)
