"""Generate tests/golden/froxelize.npz by running the REAL reference froxelizer.

Run in the build container (which has /root/reference):

    python tests/golden/make_froxelize_golden.py

Every grid written here is ``froxelpvs.froxel.froxelize`` (froxel.py:387-394,
perspective mode, froxel.py:328-348) on scenes from the reference's own scene
generator (scenegen.py:312) and on hand-built scenes that exercise the
near-plane clipper (froxel.py:203-219, 292-325): a full-cross-section quad,
quads straddling the near plane, triangles behind the origin and slivers.
The case inputs are stored as the arrays the C-ABI takes (world vertices,
triangle indices after TriScene's degenerate-triangle drop, the frustum's
origin / basis / half-extent / near / far), so the GPU box replays them
without the reference.
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
    return {m: importlib.import_module(f"froxelpvs.{m}") for m in ("core", "froxel", "scenegen")}


def _quad(z, hx, hy, cx=0.0, cy=0.0, tilt=0.0):
    """Camera-space quad centred on the forward axis at depth z; ``tilt`` varies z with y."""
    v = np.array([[cx - hx, cy - hy, z - tilt * hy], [cx + hx, cy - hy, z - tilt * hy],
                  [cx + hx, cy + hy, z + tilt * hy], [cx - hx, cy + hy, z + tilt * hy]])
    return v, np.array([[0, 1, 2], [0, 2, 3]])


def cases(m):
    core, froxel, sg = m["core"], m["froxel"], m["scenegen"]
    Vec3, Frustum, TriScene = core.Vec3, core.Frustum, core.TriScene
    out = []

    def add(name, scene, frustum, dims, ss=4, depth="linear", mode="perspective"):
        cfg = froxel.FroxelizeConfig(supersample=ss, mode=mode, depth_mode=depth)
        grid = froxel.froxelize(scene, frustum, dims, cfg)
        out.append(dict(name=name, verts=scene.vertices.copy(), tris=scene.triangles.astype(np.int64),
                        origin=frustum._o.copy(), basis=frustum._basis.copy(),
                        lens=np.array([frustum.half_extent, frustum.near, frustum.far]),
                        dims=np.array(dims), ss=np.array(ss), depth=np.array(0 if depth == "linear" else 1),
                        mode=np.array(0 if mode == "perspective" else 1), bits=grid.bits.copy()))
        print(f"{name:28s} {mode:11s} dims={dims} s={ss} {depth:6s} tris={len(scene.triangles):6d} "
              f"occupied={grid.occupied_count()}")

    # reference scene generator, viewcell frusta (SURVEY §8(f) #1 input)
    for seed, dims, ss, depth in [(0, (16, 16, 16), 4, "linear"), (1, (64, 64, 64), 4, "linear"),
                                  (2, (128, 64, 32), 2, "linear"), (3, (32, 32, 32), 1, "linear"),
                                  (4, (64, 32, 64), 3, "linear"), (5, (128, 128, 128), 4, "linear"),
                                  (6, (32, 32, 32), 4, "log")]:
        scene, cell = sg.generate_scene(sg.SceneGenConfig(seed=seed))
        add(f"scene{seed}", scene, core.build_viewcell_frustum(cell), dims, ss, depth)

    # exact frustum of the reference's tests (test_froxel.py:119-121)
    fr = Frustum(Vec3(0, 0, 0), Vec3(0, 0, 1), Vec3(0, 1, 0), Vec3(1, 0, 0), 90.0, 2.0, 18.0)
    z = fr.near + 0.5 * (fr.far - fr.near)
    v, t = _quad(z, 1.2 * z * fr.half_extent, 1.2 * z * fr.half_extent)
    add("full_span_quad", TriScene(fr._o + v @ fr._basis, t), fr, (16, 16, 16))

    # near-plane clipping: quads straddling z = near (tilted), one vertex in
    # front (1 triangle out), two in front (quad -> 2 triangles), vertex on the plane
    rng = np.random.default_rng(21)
    vs, ts = [], []
    for k in range(12):
        v, t = _quad(fr.near + rng.uniform(-0.5, 0.5), rng.uniform(0.5, 3), rng.uniform(0.5, 3),
                     rng.uniform(-2, 2), rng.uniform(-2, 2), tilt=rng.uniform(0.3, 2.0))
        ts.append(t + 4 * k)
        vs.append(v)
    vs.append(np.array([[0.0, 0.0, fr.near], [3.0, 0.0, fr.near + 4], [0.0, 3.0, fr.near - 1]]))
    ts.append(np.array([[48, 49, 50]]))
    vs.append(np.array([[-5.0, -5.0, -5.0], [5.0, -5.0, -5.0], [0.0, 5.0, -5.0]]))   # behind
    ts.append(np.array([[51, 52, 53]]))
    vs.append(np.array([[1.0, 1.0, 30.0], [2.0, 1.0, 30.0], [1.0, 2.0, 30.0]]))      # beyond far
    ts.append(np.array([[54, 55, 56]]))
    vs.append(np.array([[0.0, 0.0, 5.0], [1e-7, 0.0, 5.0], [0.0, 4.0, 9.0]]))        # sliver
    ts.append(np.array([[57, 58, 59]]))
    verts = np.concatenate(vs)
    add("near_clip", TriScene(fr._o + verts @ fr._basis, np.concatenate(ts)), fr, (32, 32, 32), 4)

    # random triangle soup around a rotated viewcell frustum, many near-plane crossings
    cell = core.ViewCell.from_forward(Vec3(0.3, 1.2, -0.4), 0.3, 60.0, 15.0,
                                      Vec3(0.6, 0.1, 0.8), 0.3, 20.0)
    fr2 = core.build_viewcell_frustum(cell)
    c = rng.uniform(-6, 6, size=(400, 1, 3)) + fr2._o
    soup = c + rng.normal(scale=1.5, size=(400, 3, 3))
    add("soup", TriScene(soup.reshape(-1, 3), np.arange(1200).reshape(-1, 3)), fr2, (64, 48, 40), 4)
    add("soup_s1", TriScene(soup.reshape(-1, 3), np.arange(1200).reshape(-1, 3)), fr2, (64, 48, 40), 1)

    # empty scene
    add("empty", TriScene(np.zeros((0, 3)), np.zeros((0, 3), dtype=np.int64)), fr, (16, 16, 16))

    # orthographic three-view mode (froxel.py:351-376), the dataset generator's default
    for seed, dims, ss, depth in [(0, (16, 16, 16), 4, "linear"), (1, (64, 64, 64), 2, "linear"),
                                  (2, (32, 16, 24), 3, "linear"), (3, (32, 32, 32), 1, "log")]:
        scene, cell = sg.generate_scene(sg.SceneGenConfig(seed=seed))
        add(f"ortho_scene{seed}", scene, core.build_viewcell_frustum(cell), dims, ss, depth, mode="ortho")
    v, t = _quad(z, 1.2 * z * fr.half_extent, 1.2 * z * fr.half_extent)
    add("ortho_full_span_quad", TriScene(fr._o + v @ fr._basis, t), fr, (16, 16, 16), mode="ortho")
    add("ortho_soup", TriScene(soup.reshape(-1, 3), np.arange(1200).reshape(-1, 3)), fr2, (64, 48, 40), 2,
        mode="ortho")
    add("ortho_empty", TriScene(np.zeros((0, 3)), np.zeros((0, 3), dtype=np.int64)), fr, (16, 16, 16), mode="ortho")
    return out


def main():
    m = _ref()
    arrays = {}
    cs = cases(m)
    for i, c in enumerate(cs):
        for k, v in c.items():
            arrays[f"c{i}_{k}"] = np.array(v) if k == "name" else v
    arrays["ncases"] = np.array(len(cs))
    path = os.path.join(HERE, "froxelize.npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


if __name__ == "__main__":
    main()
