"""dataset.generate_dataset (device froxelize + GT PVS) vs the reference's
scenegen.py:394-431 on the same scenes: every FPVS file and the manifest are
byte-identical (tests/golden/dataset.npz, tests/golden/make_dataset_golden.py)."""

from __future__ import annotations

import os
from types import SimpleNamespace

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "dataset.npz")


def _golden():
    return np.load(GOLDEN)


def test_frame_seed_matches_reference():
    from paper_2509_24677_b200.dataset import frame_seed
    g = _golden()
    master, n = int(g["params"][0]), int(g["params"][1])
    for i in range(n):
        assert frame_seed(master, i) == int(g[f"f{i}_seed"])


def _scene_fn(g):
    from paper_2509_24677_b200 import views
    by_seed = {}
    for i in range(int(g["params"][1])):
        cl = g[f"f{i}_cell"]
        cell = views.ViewCell(tuple(cl[0:3]), cl[3], cl[4], cl[5], tuple(cl[6:9]), tuple(cl[9:12]),
                              tuple(cl[12:15]), cl[15], cl[16])
        scene = SimpleNamespace(vertices=g[f"f{i}_verts"], triangles=g[f"f{i}_tris"],
                                primitive_ids=g[f"f{i}_prim_ids"])
        by_seed[int(g[f"f{i}_seed"])] = (scene, cell)
    return lambda seed: by_seed[int(seed)]


@pytest.mark.gpu
def test_generate_dataset_byte_identical(tmp_path):
    from paper_2509_24677_b200.dataset import generate_dataset
    from paper_2509_24677_b200.froxelize import FroxelizeConfig
    from paper_2509_24677_b200.gtpvs import OracleConfig
    g = _golden()
    master, n, nx, ny, nz, views_n, ss = (int(v) for v in g["params"])
    manifest = generate_dataset(_scene_fn(g), master, n, tmp_path, dims=(nx, ny, nz),
                                ocfg=OracleConfig(viewpoints=views_n),
                                fcfg=FroxelizeConfig(supersample=ss, mode="ortho"))
    assert manifest.read_bytes() == g["manifest"].tobytes()
    for i in range(n):
        for kind in ("geometry", "gt"):
            got = (tmp_path / f"{kind}_{i:05d}.fpvs").read_bytes()
            assert got == g[f"f{i}_{kind}"].tobytes(), (i, kind)


@pytest.mark.gpu
def test_pair_producer_subset_and_device_buffers():
    import torch
    from paper_2509_24677_b200.dataset import PairProducer
    from paper_2509_24677_b200.froxelize import FroxelizeConfig
    from paper_2509_24677_b200.gtpvs import OracleConfig
    g = _golden()
    master, n, nx, ny, nz, views_n, ss = (int(v) for v in g["params"])
    scene, cell = _scene_fn(g)(int(g["f0_seed"]))
    prod = PairProducer((nx, ny, nz), OracleConfig(viewpoints=views_n), FroxelizeConfig(supersample=ss, mode="ortho"))
    geo, gt, ok = prod.pair(scene, cell)
    assert geo.is_cuda and gt.is_cuda and bool(ok)
    assert int(torch.count_nonzero(gt & ~geo)) == 0
    # the FPVS payload is the packed grid after the header
    nbytes = nx * ny * nz // 8
    assert np.array_equal(geo.cpu().numpy(), g["f0_geometry"][-nbytes:])
    assert np.array_equal(gt.cpu().numpy(), g["f0_gt"][-nbytes:])
