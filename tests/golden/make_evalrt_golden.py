"""Generate tests/golden/evalrt.npz by running the REAL reference consumers.

Run in the build container (which has /root/reference):

    python tests/golden/make_evalrt_golden.py

Per case (reference scene-generator scenes and its own test scenes): the
froxel -> primitive-id map of ``froxel_id_map`` (froxel.py:397-417) as
sorted (x, y, z, id) rows, ``cull`` (evalrt.py:62-68) for random PVS grids,
``render_depth`` (oracle.py:107-138) depth / id buffers for two cameras,
``pixel_error_rate`` (evalrt.py:71-84) and ``far_field_merge``
(evalrt.py:87-106), and ``froxel_metrics`` counts (evalrt.py:38-59).
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
    return {m: importlib.import_module(f"froxelpvs.{m}") for m in ("core", "froxel", "oracle", "scenegen", "evalrt")}


def _cam_row(c):
    return np.concatenate([c.position.as_array(), c.right.as_array(), c.up.as_array(), c.forward.as_array(),
                           [c.half_extent, c.near, c.far], [c.fov_deg]])


def _cell_row(cell):
    return np.concatenate([cell.center.as_array(), [cell.radius, cell.fov_deg, cell.beta_deg],
                           cell.forward.as_array(), cell.up.as_array(), cell.right.as_array(), [cell.near, cell.far]])


def cases(m):
    core, froxel, oracle, sg, ev = m["core"], m["froxel"], m["oracle"], m["scenegen"], m["evalrt"]
    rng = np.random.default_rng(31)
    out = []
    # the last two use the orthographic fragment stream, as the reference's
    # CLI infer / metrics path does (cli.py:297-300)
    for seed, dims, ss, count, mode in [(0, (16, 16, 16), 4, (6, 14), "perspective"),
                                        (1, (32, 16, 24), 2, (3, 6), "perspective"),
                                        (2, (32, 32, 32), 4, (6, 14), "perspective"),
                                        (3, (16, 16, 16), 4, (6, 14), "ortho"),
                                        (4, (32, 24, 16), 2, (3, 6), "ortho")]:
        scene, cell = sg.generate_scene(sg.SceneGenConfig(seed=seed, count_range=count))
        fr = core.build_viewcell_frustum(cell)
        cfg = froxel.FroxelizeConfig(supersample=ss, mode=mode)
        idm = froxel.froxel_id_map(scene, fr, dims, cfg)
        rows = np.array(sorted((x, y, z, p) for (x, y, z), ids in idm.items() for p in ids), dtype=np.int64)
        geo = froxel.froxelize(scene, fr, dims, cfg)
        pvs_list, culls = [], []
        for k, dens in enumerate((0.02, 0.2, 1.0)):
            dense = rng.random(dims) < dens
            pvs = froxel.FroxelGrid.from_dense(dense)
            pvs_list.append(pvs.bits.copy())
            culls.append(np.array(sorted(ev.cull(scene, pvs, idm)), dtype=np.int64))
        gt = oracle.compute_gt_pvs(scene, cell, dims, oracle.OracleConfig(viewpoints=8))
        cams = oracle.sample_viewpoints(cell, oracle.OracleConfig(viewpoints=8))[:2]
        res = (48, 40)
        bufs = [oracle.render_depth(scene, c, res) for c in cams]
        per = ev.pixel_error_rate(scene, cams[0], gt, idm, resolution=res)
        thr = 0.5 * (cell.near + cell.far)
        ff = np.array(sorted(ev.far_field_merge(scene, cell, gt, idm, thr, resolution=res)), dtype=np.int64)
        met = ev.froxel_metrics(froxel.FroxelGrid(dims, bits=pvs_list[1]), gt)
        c = dict(name=np.array(f"scene{seed}" + ("_ortho" if mode == "ortho" else "")),
                 mode=np.array(0 if mode == "perspective" else 1), verts=scene.vertices.copy(), tris=scene.triangles.astype(np.int64),
                 prim_ids=scene.primitive_ids.astype(np.int64), cell=_cell_row(cell),
                 frustum=np.concatenate([fr._o, fr._basis.reshape(-1), [fr.half_extent, fr.near, fr.far]]),
                 dims=np.array(dims), ss=np.array(ss), idmap=rows, geo=geo.bits.copy(), gt=gt.bits.copy(),
                 pvs=np.stack(pvs_list), cams=np.stack([_cam_row(x) for x in cams]), res=np.array(res),
                 depth=np.stack([b.depth for b in bufs]), prim=np.stack([b.prim for b in bufs]), per=np.array(per),
                 ff_threshold=np.array(thr), ff=ff,
                 metrics=np.array([met.tp, met.fp, met.fn, met.gtp]), rates=np.array([met.fnr, met.fpr]))
        for k, cl in enumerate(culls):
            c[f"cull{k}"] = cl
        out.append(c)
        print(f"scene{seed} dims={dims} tris={len(scene.triangles)} idmap rows={len(rows)} culls="
              f"{[len(x) for x in culls]} per={per:.4f} far-field={len(ff)}")
    return out


def main():
    m = _ref()
    arrays = {}
    cs = cases(m)
    for i, c in enumerate(cs):
        for k, v in c.items():
            arrays[f"c{i}_{k}"] = v
    arrays["ncases"] = np.array(len(cs))
    path = os.path.join(HERE, "evalrt.npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


if __name__ == "__main__":
    main()
