"""Generate tests/golden/dataset.npz by running the REAL reference dataset loop.

Run in the build container (which has /root/reference):

    python tests/golden/make_dataset_golden.py

``generate_dataset`` (scenegen.py:394-431) writes 3 frames at 16x24x16
(ortho froxelize, 16 uniform-grid viewpoints) into a temp dir; the npz keeps
every file's bytes (FPVS grids + manifest) and, per frame, the scene and
viewcell ``generate_scene`` made for that frame's seed, so the GPU box can
replay the same scenes through ``dataset.generate_dataset`` without the
reference.
"""

from __future__ import annotations

import os
import sys
import tempfile
from dataclasses import replace

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = os.environ.get("FPVS_REFERENCE_SRC", "/root/reference/pkg/src")
MASTER_SEED, N_FRAMES, DIMS, VIEWPOINTS, SS = 11, 3, (16, 24, 16), 16, 2


def _cell_row(cell):
    return np.concatenate([cell.center.as_array(), [cell.radius, cell.fov_deg, cell.beta_deg],
                           cell.forward.as_array(), cell.up.as_array(), cell.right.as_array(), [cell.near, cell.far]])


def main():
    if not os.path.isdir(os.path.join(REF_SRC, "froxelpvs")):
        raise SystemExit("reference not found at " + REF_SRC)
    sys.path.insert(0, REF_SRC)
    from froxelpvs import froxel, oracle, scenegen as sg
    cfg = sg.SceneGenConfig(seed=MASTER_SEED, count_range=(4, 9))
    ocfg = oracle.OracleConfig(viewpoints=VIEWPOINTS)
    fcfg = froxel.FroxelizeConfig(supersample=SS, mode="ortho")
    arrays = {}
    with tempfile.TemporaryDirectory() as d:
        manifest = sg.generate_dataset(cfg, N_FRAMES, d, dims=DIMS, ocfg=ocfg, fcfg=fcfg)
        arrays["manifest"] = np.frombuffer(manifest.read_bytes(), dtype=np.uint8)
        for i in range(N_FRAMES):
            seed = sg.frame_seed(cfg.seed, i)
            scene, cell = sg.generate_scene(replace(cfg, seed=seed))
            arrays[f"f{i}_seed"] = np.array(seed, dtype=np.uint64)
            arrays[f"f{i}_verts"] = scene.vertices.copy()
            arrays[f"f{i}_tris"] = scene.triangles.astype(np.int64)
            arrays[f"f{i}_prim_ids"] = scene.primitive_ids.astype(np.int64)
            arrays[f"f{i}_cell"] = _cell_row(cell)
            for kind in ("geometry", "gt"):
                arrays[f"f{i}_{kind}"] = np.fromfile(os.path.join(d, f"{kind}_{i:05d}.fpvs"), dtype=np.uint8)
            print(f"frame {i} seed {seed} tris {len(scene.triangles)}")
    arrays["params"] = np.array([MASTER_SEED, N_FRAMES, *DIMS, VIEWPOINTS, SS], dtype=np.int64)
    path = os.path.join(HERE, "dataset.npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


if __name__ == "__main__":
    main()
