"""Device consumers of the PVS (evalrt.py) vs the reference.

Pinned on tests/golden/evalrt.npz (tests/golden/make_evalrt_golden.py): the
reference's own froxel_id_map (froxel.py:397-417), cull (evalrt.py:62-68),
render_depth (oracle.py:107-138), pixel_error_rate (evalrt.py:71-84),
far_field_merge (evalrt.py:87-106) and froxel_metrics (evalrt.py:38-59)
outputs, over both fragment streams (perspective and the CLI's ortho).  All
comparisons are exact (sets, ids, float64 depths, the PER
fraction).
"""

from __future__ import annotations

import os
from types import SimpleNamespace

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "evalrt.npz")


def _cases():
    g = np.load(GOLDEN)
    out = []
    for i in range(int(g["ncases"])):
        p = f"c{i}_"
        out.append({k[len(p):]: g[k] for k in g.files if k.startswith(p)})
    return out


CASES = _cases()
IDS = [str(c["name"]) for c in CASES]


def _objs(c):
    from paper_2509_24677_b200 import views
    from paper_2509_24677_b200.froxelize import FroxelizeConfig, Frustum
    scene = SimpleNamespace(vertices=c["verts"], triangles=c["tris"], primitive_ids=c["prim_ids"])
    f = c["frustum"]
    fr = Frustum(f[0:3], f[3:12], f[12], f[13], f[14])
    cl = c["cell"]
    cell = views.ViewCell(tuple(cl[0:3]), cl[3], cl[4], cl[5], tuple(cl[6:9]), tuple(cl[9:12]), tuple(cl[12:15]),
                          cl[15], cl[16])
    cams = [views.Camera(tuple(r[0:3]), tuple(r[9:12]), tuple(r[6:9]), tuple(r[3:6]), r[15], r[13], r[14])
            for r in c["cams"]]
    mode = "ortho" if int(c.get("mode", 0)) == 1 else "perspective"
    return scene, fr, cell, cams, tuple(int(x) for x in c["dims"]), FroxelizeConfig(supersample=int(c["ss"]),
                                                                                    mode=mode)


@pytest.mark.parametrize("idx", range(len(CASES)), ids=IDS)
def test_id_map_and_cull(idx):
    from paper_2509_24677_b200 import evalrt
    from paper_2509_24677_b200.froxel import FroxelGrid
    c = CASES[idx]
    scene, fr, _, _, dims, cfg = _objs(c)
    idm = evalrt.froxel_id_map(scene, fr, dims, cfg)
    for k in range(3):
        got = sorted(evalrt.cull(scene, FroxelGrid(dims, bits=c["pvs"][k]), idm))
        assert got == c[f"cull{k}"].tolist(), k
    rows = sorted((x, y, z, p) for (x, y, z), ids in idm.items() for p in ids)
    assert np.array_equal(np.array(rows, dtype=np.int64).reshape(-1, 4), c["idmap"])
    # key set == froxelized occupancy (test_froxel.py:236-245)
    occ = FroxelGrid(dims, bits=c["geo"]).to_dense()
    assert set(idm.keys()) == set(map(tuple, np.argwhere(occ).tolist()))


@pytest.mark.parametrize("idx", range(len(CASES)), ids=IDS)
def test_render_depth_per_far_field_metrics(idx):
    from paper_2509_24677_b200 import evalrt
    from paper_2509_24677_b200.froxel import FroxelGrid
    c = CASES[idx]
    scene, fr, cell, cams, dims, cfg = _objs(c)
    res = tuple(int(x) for x in c["res"])
    for k, cam in enumerate(cams):
        buf = evalrt.render_depth(scene, cam, res)
        assert np.array_equal(buf.prim, c["prim"][k])
        assert np.array_equal(buf.depth, c["depth"][k])
    idm = evalrt.froxel_id_map(scene, fr, dims, cfg)
    gt = FroxelGrid(dims, bits=c["gt"])
    assert evalrt.pixel_error_rate(scene, cams[0], gt, idm, resolution=res) == float(c["per"])
    ff = evalrt.far_field_merge(scene, cell, gt, idm, float(c["ff_threshold"]), resolution=res)
    assert sorted(ff) == c["ff"].tolist()
    met = evalrt.froxel_metrics(FroxelGrid(dims, bits=c["pvs"][1]), gt)
    assert [met.tp, met.fp, met.fn, met.gtp] == c["metrics"].tolist()
    assert [met.fnr, met.fpr] == c["rates"].tolist()


def test_cull_everything_and_nothing():
    """An all-ones PVS keeps exactly the primitives with a fragment; an empty one keeps none."""
    from paper_2509_24677_b200 import evalrt
    from paper_2509_24677_b200.froxel import FroxelGrid
    c = CASES[0]
    scene, fr, _, _, dims, cfg = _objs(c)
    idm = evalrt.froxel_id_map(scene, fr, dims, cfg)
    full = FroxelGrid(dims, bits=np.full(int(np.prod(dims)) // 8, 0xFF, np.uint8))
    assert evalrt.cull(scene, full, idm) == set().union(*idm.values())
    assert evalrt.cull(scene, FroxelGrid(dims), idm) == set()
