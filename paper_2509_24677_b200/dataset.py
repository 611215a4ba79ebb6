"""Training-pair producer on the device: scenegen.py:394-431 ``generate_dataset``
around the device froxelizer and GT PVS (SURVEY.md §3.4, §8(f) #1 + #3).

Per frame the reference froxelizes the scene into the viewcell frustum
(``FroxelizeConfig(mode="ortho")`` by default), computes the GT PVS with
``geometry=`` so every GT fragment is OR-ed into the geometry (GT ⊆ geometry
holds bit-exactly), checks the subset property and writes both grids as FPVS
files plus a line-oriented manifest.  Here both grids are produced on the
device (``fpvs_froxelize_ortho`` / ``fpvs_froxelize`` then ``fpvs_gt_pvs``
with the geometry buffer), the subset check is one device reduction, and
``PairProducer.pair`` hands the packed grids to the trainer without a host
hop.  The scene generator itself stays out of scope: the
caller passes ``scene_fn(seed) -> (scene, cell)`` — the reference's
``lambda s: generate_scene(replace(cfg, seed=s))`` fits unchanged.
"""

from __future__ import annotations

from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _lib, views
from .froxel import FroxelGrid
from .froxelize import FroxelizeConfig, Froxelizer
from .gtpvs import GtPvs, OracleConfig


def _torch():
    import torch
    return torch


@dataclass(frozen=True)
class FrameRecord:
    """scenegen.py:375-379."""
    index: int
    seed: int
    geometry_path: str
    gt_path: str


class DatasetError(RuntimeError):
    """scenegen.py:382-385: a frame failed validation or could not be written."""

    def __init__(self, index: int, message: str):
        super().__init__(f"frame {index}: {message}")
        self.index = index


def frame_seed(master_seed: int, index: int) -> int:
    """Stable per-frame seed (scenegen.py:388-391): the first 64-bit word of
    ``SeedSequence([master_seed, index])``."""
    ss = np.random.SeedSequence([int(master_seed), int(index)])
    return int(ss.generate_state(1, np.uint64)[0])


class PairProducer:
    """(geometry, GT PVS) packed grids of one scene + viewcell, on the device."""

    def __init__(self, dims=(32, 32, 32), ocfg: OracleConfig | None = None, fcfg: FroxelizeConfig | None = None,
                 device="cuda"):
        _lib.require_cuda()
        self.dims = tuple(int(d) for d in dims)
        if self.dims[0] % 8:
            raise ValueError(f"N_x must be divisible by 8, got {self.dims[0]}")
        self.ocfg = ocfg or OracleConfig()
        self.fcfg = fcfg or FroxelizeConfig(mode="ortho")
        self.device = device
        nbytes = int(np.prod(self.dims)) // 8
        self.padded = (nbytes + 3) & ~3
        self.nbytes = nbytes

    def pair(self, scene, cell):
        """Device uint8 tensors (geometry, gt), each Nx*Ny*Nz/8 bytes, and the
        subset flag (device bool): froxelize, then compute_gt_pvs(geometry=...)
        as scenegen.py:415-418."""
        torch = _torch()
        geo = torch.zeros(self.padded, dtype=torch.uint8, device=self.device)
        gt = torch.zeros(self.padded, dtype=torch.uint8, device=self.device)
        frustum = views.build_viewcell_frustum(cell)
        Froxelizer(scene.vertices, scene.triangles, self.device).run(frustum, self.dims, self.fcfg,
                                                                      out=geo[:self.nbytes])
        g = GtPvs(scene.vertices, scene.triangles, getattr(scene, "primitive_ids", None), self.device)
        g.for_cell(cell, self.dims, self.ocfg, self.fcfg, out=gt, geometry=geo)
        ok = ~torch.any(gt & ~geo)
        return geo[:self.nbytes], gt[:self.nbytes], ok


def generate_dataset(scene_fn, master_seed: int, n_frames: int, out_dir, dims=(32, 32, 32),
                     ocfg: OracleConfig | None = None, fcfg: FroxelizeConfig | None = None) -> Path:
    """scenegen.py:394-431 with the grids computed on the device.

    ``scene_fn(seed) -> (scene, cell)`` stands in for
    ``generate_scene(replace(cfg, seed=seed))``; ``master_seed`` is
    ``cfg.seed``.  Writes ``geometry_%05d.fpvs`` / ``gt_%05d.fpvs`` and
    ``manifest.txt`` (``index seed geometry gt`` lines) byte-identical to the
    reference's for the same scenes."""
    out_dir = Path(out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    prod = PairProducer(dims, ocfg, fcfg)
    lines = ["# froxelpvs dataset: index seed geometry gt"]
    for i in range(n_frames):
        seed = frame_seed(master_seed, i)
        scene, cell = scene_fn(seed)
        geo_d, gt_d, ok = prod.pair(scene, cell)
        if not bool(ok):
            raise DatasetError(i, "ground truth escapes the geometry grid")
        ss = prod.fcfg.supersample
        geometry = FroxelGrid(prod.dims, role="geometry", supersample=ss, bits=geo_d.cpu().numpy())
        gt = FroxelGrid(prod.dims, role="gt_pvs", supersample=ss, bits=gt_d.cpu().numpy())
        geo_name, gt_name = f"geometry_{i:05d}.fpvs", f"gt_{i:05d}.fpvs"
        try:
            geometry.save(out_dir / geo_name)
            gt.save(out_dir / gt_name)
        except OSError as exc:
            raise DatasetError(i, f"write failed: {exc}") from exc
        lines.append(f"{i} {seed} {geo_name} {gt_name}")
    manifest = out_dir / "manifest.txt"
    try:
        manifest.write_text("\n".join(lines) + "\n")
    except OSError as exc:
        raise DatasetError(n_frames, f"manifest write failed: {exc}") from exc
    return manifest
