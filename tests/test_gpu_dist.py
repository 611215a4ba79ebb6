"""Data-parallel training on the device: ``train()`` with 2 ranks (gloo with
CUDA tensors, both ranks on GPU 0 — the collective is host-mediated, so no
kernel waits on another rank) equals single-rank ``train()`` on the full
batch, the reference's batch-mean semantics (neural.py:472-481) for even and
uneven shards; one exchange (all-reduce) per step carries the gradient, the
loss and the hard counts; a non-finite loss raises TrainingDiverged."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from paper_2509_24677_b200 import synth
from paper_2509_24677_b200.froxel import FroxelGrid

pytestmark = pytest.mark.gpu

DIMS = (32, 32, 16)


def _pairs(n):
    out = []
    for s in range(n):
        occ = synth.box_grid(DIMS, 30, 1, 4, 70 + s)
        out.append((FroxelGrid.from_dense(occ), FroxelGrid.from_dense(synth.first_hit_labels(occ), role="gt_pvs")))
    return out


def _cfg():
    from paper_2509_24677_b200.neural import TrainConfig
    return TrainConfig(lr=1e-2, epochs=2, batch_size=3, seed=4)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from paper_2509_24677_b200.neural import ModelConfig
    from paper_2509_24677_b200.train import train
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    calls = {"n": 0}
    orig = dist.all_reduce

    def counting(*a, **k):
        calls["n"] += 1
        return orig(*a, **k)
    dist.all_reduce = counting
    try:
        net, hist = train(_pairs(5), ModelConfig.config1(), _cfg())
        w = [L.w.cpu().numpy().copy() for L in net.layers] + [L.b.cpu().numpy().copy() for L in net.layers]
        q.put((rank, w, hist, calls["n"]))
    finally:
        dist.all_reduce = orig
        dist.destroy_process_group()


def test_two_rank_train_equals_single_rank():
    import torch.multiprocessing as mp
    from paper_2509_24677_b200.neural import ModelConfig
    from paper_2509_24677_b200.train import train
    net, hist = train(_pairs(5), ModelConfig.config1(), _cfg())
    want = [L.w.cpu().numpy() for L in net.layers] + [L.b.cpu().numpy() for L in net.layers]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        r, w, h, n = q.get(timeout=300)
        res[r] = (w, h, n)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    steps = 2 * 2  # 2 epochs x ceil(5 / 3) batches (a 2 + 1 split of 3, then 1 + 1 of 2)
    for r in range(2):
        w, h, n = res[r]
        assert n == steps, f"rank {r}: {n} all-reduces for {steps} steps"
        for a, b in zip(w, want):
            assert np.abs(a - b).max() <= 1e-6 * max(1.0, float(np.abs(b).max()))
        for he, hw in zip(h, hist):
            assert abs(he["loss"] - hw["loss"]) <= 1e-6
            assert he["fnr"] == hw["fnr"] and he["fpr"] == hw["fpr"]


def test_non_finite_loss_raises_training_diverged():
    from paper_2509_24677_b200.neural import ModelConfig, TrainConfig, TrainingDiverged
    from paper_2509_24677_b200.train import train
    with pytest.raises(TrainingDiverged) as ei:
        train(_pairs(3), ModelConfig.config1(), TrainConfig(lr=1e38, epochs=3, batch_size=1, seed=1))
    assert ei.value.batch_index >= 1
