"""Generate tests/golden/gtpvs.npz by running the REAL reference GT-PVS generator.

Run in the build container (which has /root/reference):

    python tests/golden/make_gtpvs_golden.py

Every grid written here is ``froxelpvs.oracle.compute_gt_pvs``
(oracle.py:141-172) — depth-buffer rendering per sampled viewpoint
(oracle.py:107-138), reprojection into the viewcell frustum (core.py:380-452)
— on the reference's scene-generator scenes and on hand-built scenes (a full
occluder, negative primitive ids, the empty scene).  Stored per case: the
scene arrays, the cell, the viewpoint settings, the cameras the reference
sampled (pinning ``views.sample_viewpoints``), the viewcell frustum, dims,
depth-buffer resolution, depth mode, the GT bits and, when the case passes a
geometry grid, that grid before and after (compute_gt_pvs ORs into it).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = os.environ.get("FPVS_REFERENCE_SRC", "/root/reference/pkg/src")


def _ref():
    if not os.path.isdir(os.path.join(REF_SRC, "froxelpvs")):
        raise SystemExit("reference not found at " + REF_SRC)
    sys.path.insert(0, REF_SRC)
    import importlib
    return {m: importlib.import_module(f"froxelpvs.{m}") for m in ("core", "froxel", "oracle", "scenegen")}


def _cam_row(c):
    return np.concatenate([c.position.as_array(), c.right.as_array(), c.up.as_array(), c.forward.as_array(),
                           [c.half_extent, c.near, c.far]])


def _cell_row(cell):
    return np.concatenate([cell.center.as_array(), [cell.radius, cell.fov_deg, cell.beta_deg],
                           cell.forward.as_array(), cell.up.as_array(), cell.right.as_array(), [cell.near, cell.far]])


def cases(m):
    core, froxel, oracle, sg = m["core"], m["froxel"], m["oracle"], m["scenegen"]
    Vec3, TriScene = core.Vec3, core.TriScene
    out = []

    def add(name, scene, cell, dims, viewpoints=8, mode="uniform-grid", seed=0, res=None, depth="linear",
            cams=None, geometry=None):
        ocfg = oracle.OracleConfig(viewpoints=viewpoints, mode=mode, seed=seed, depth_resolution=res)
        fcfg = froxel.FroxelizeConfig(depth_mode=depth)
        used = cams if cams is not None else oracle.sample_viewpoints(cell, ocfg)
        geo_in = None if geometry is None else geometry.bits.copy()
        gt = oracle.compute_gt_pvs(scene, cell, dims, ocfg, fcfg, geometry=geometry, cameras=cams)
        fr = core.build_viewcell_frustum(cell)
        c = dict(name=np.array(name), verts=scene.vertices.copy(), tris=scene.triangles.astype(np.int64),
                 prim_ids=scene.primitive_ids.astype(np.int64), cell=_cell_row(cell),
                 sampling=np.array([viewpoints, 0 if mode == "uniform-grid" else 1, seed,
                                    -1 if cams is None else len(cams)]),
                 cams=np.stack([_cam_row(x) for x in used]) if used else np.zeros((0, 15)),
                 frustum=np.concatenate([fr._o, fr._basis.reshape(-1), [fr.half_extent, fr.near, fr.far]]),
                 dims=np.array(dims), res=np.array(ocfg.resolution_for(dims)),
                 depth=np.array(0 if depth == "linear" else 1), bits=gt.bits.copy())
        if geo_in is not None:
            c["geo_in"] = geo_in
            c["geo_out"] = geometry.bits.copy()
        out.append(c)
        print(f"{name:22s} dims={dims} M={len(used):3d} res={ocfg.resolution_for(dims)} {depth:6s} "
              f"tris={len(scene.triangles):5d} gt={gt.occupied_count()}")

    for seed, dims, vp, mode, res, depth in [(0, (16, 16, 16), 8, "uniform-grid", None, "linear"),
                                             (1, (32, 32, 32), 16, "uniform-grid", None, "linear"),
                                             (2, (64, 32, 48), 6, "uniform-random", (320, 160), "linear"),
                                             (3, (32, 32, 32), 8, "uniform-grid", None, "log"),
                                             (4, (32, 16, 24), 1, "uniform-grid", None, "linear")]:
        scene, cell = sg.generate_scene(sg.SceneGenConfig(seed=seed))
        add(f"scene{seed}", scene, cell, dims, vp, mode, 5, res, depth)

    # geometry OR (oracle.py:164-170): the perspective froxelization as input
    scene, cell = sg.generate_scene(sg.SceneGenConfig(seed=7))
    fr = core.build_viewcell_frustum(cell)
    geo = froxel.froxelize(scene, fr, (32, 32, 32), froxel.FroxelizeConfig())
    add("scene7_geometry", scene, cell, (32, 32, 32), 12, geometry=geo)

    # explicit camera subset (test_oracle.py:141-148)
    scene, cell = sg.generate_scene(sg.SceneGenConfig(seed=4, count_range=(3, 6)))
    cams = oracle.sample_viewpoints(cell, oracle.OracleConfig(viewpoints=24))
    add("cams_subset", scene, cell, (16, 16, 16), 24, cams=cams[:8])

    # full occluder at layer 8.5/16 (test_oracle.py:113-137)
    cell = core.ViewCell.from_forward(Vec3(0.0, 1.5, 0.0), 0.3, 60.0, 15.0, Vec3(0.0, 0.0, 1.0), 0.3, 20.0)
    fr = core.build_viewcell_frustum(cell)
    z = fr.near + 8.5 / 16.0 * (fr.far - fr.near)
    half = 1.5 * z * fr.half_extent
    q = np.array([[-half, -half], [half, -half], [half, half], [-half, half]])
    qt = np.array([[0, 1, 2], [0, 2, 3]])
    occ = fr._o + np.column_stack([q[:, 0], q[:, 1], np.full(4, z)]) @ fr._basis
    bz = fr.near + 0.9 * (fr.far - fr.near)
    beh = fr._o + np.column_stack([q[:, 0], q[:, 1], np.full(4, bz)]) @ fr._basis
    add("occluder", TriScene(np.vstack([occ, beh]), np.vstack([qt, qt + 4])), cell, (16, 16, 16), 32)

    # negative primitive ids: pixels whose nearest fragment has id < 0 are not fragments
    scene, cell = sg.generate_scene(sg.SceneGenConfig(seed=9, count_range=(3, 5)))
    pids = np.arange(len(scene.triangles)) - len(scene.triangles) // 3
    neg = TriScene(scene.vertices, scene.triangles, primitive_ids=pids)
    add("negative_ids", neg, cell, (32, 32, 32), 8)

    add("empty", TriScene(np.zeros((0, 3)), np.zeros((0, 3), dtype=np.int64)), cell, (16, 16, 16), 8)
    return out


def main():
    m = _ref()
    arrays = {}
    cs = cases(m)
    for i, c in enumerate(cs):
        for k, v in c.items():
            arrays[f"c{i}_{k}"] = v
    arrays["ncases"] = np.array(len(cs))
    path = os.path.join(HERE, "gtpvs.npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


if __name__ == "__main__":
    main()
