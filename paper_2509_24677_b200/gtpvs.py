"""Device ground-truth PVS: drop-in for oracle.py:141-172.

``compute_gt_pvs(scene, cell, dims, ocfg, fcfg, geometry, cameras)`` keeps the
reference's signature and result (a ``FroxelGrid`` with role ``gt_pvs``;
``geometry``, when given, gets every GT bit OR-ed in).  The cameras are
sampled on the host by ``views.sample_viewpoints`` (bit-identical to the
reference's), the work runs in ``fpvs_gt_pvs`` (csrc/froxelize.cu): all
cameras' depth buffers are rasterized in one pass over the flat
(camera, triangle, sample) space, z-tested with 64-bit atomics, then every
covered pixel is reprojected into the viewcell frustum.  No CPU path.

``GtPvs`` keeps the scene resident for many viewcells (the dataset loop of
scenegen.py:394-431) and writes device grids that feed training directly.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib, views
from .froxel import FroxelGrid
from .froxelize import FroxelizeConfig, Frustum

# depth buffers + slots of one camera batch are kept under this many bytes
WORKSPACE_BUDGET = 6 << 30


def _torch():
    import torch
    return torch


@dataclass
class OracleConfig:
    """Mirror of oracle.py:24-45."""

    viewpoints: int = 128
    mode: str = "uniform-grid"
    seed: int = 0
    depth_resolution: tuple | None = None

    def __post_init__(self):
        if self.viewpoints < 1:
            raise ValueError("viewpoint count must be >= 1")
        if self.mode not in ("uniform-grid", "uniform-random"):
            raise ValueError(f"unknown sampling mode {self.mode!r}")

    def resolution_for(self, dims) -> tuple:
        if self.depth_resolution is not None:
            w, h = self.depth_resolution
            if w < dims[0] or h < dims[1]:
                raise ValueError("depth buffer must be at least the grid cross-section")
            return int(w), int(h)
        return 4 * int(dims[0]), 4 * int(dims[1])


def _cam_rows(cams) -> np.ndarray:
    """(M, 15) float64 fpvs_frustum rows: position, right, up, forward, half_extent, near, far."""
    rows = []
    for c in cams:
        c = c if isinstance(c, views.Camera) else views.Camera.of(c)
        rows.append(np.concatenate([c.position, c.right, c.up, c.forward, [c.half_extent, c.near, c.far]]))
    return np.asarray(rows, dtype=np.float64).reshape(-1, 15)


class GtPvs:
    """A triangle scene resident on the device; GT PVS grids for any viewcell."""

    def __init__(self, vertices, triangles, primitive_ids=None, device="cuda"):
        torch = _torch()
        _lib.require_cuda()
        v = np.asarray(vertices, dtype=np.float64).reshape(-1, 3)
        t = np.asarray(triangles, dtype=np.int64).reshape(-1, 3)
        if t.size and (t.min() < 0 or t.max() >= len(v)):
            raise ValueError("triangle index out of range")
        self.verts = torch.from_numpy(np.ascontiguousarray(v)).to(device)
        self.tris = torch.from_numpy(np.ascontiguousarray(t)).to(device)
        self.prim = None
        if primitive_ids is not None:
            pids = np.asarray(primitive_ids, dtype=np.int64).reshape(-1)
            if len(pids) != len(t):
                raise ValueError("primitive_ids must have one entry per triangle")
            if (pids < 0).any():  # ids only matter when a negative one can win a pixel
                self.prim = torch.from_numpy(np.ascontiguousarray(pids)).to(device)
        self.device = device
        self._ws = None

    @property
    def ntris(self) -> int:
        return int(self.tris.shape[0])

    def _ws_for(self, ncams, res):
        torch = _torch()
        need = _lib.size("fpvs_gt_pvs_workspace_size", self.ntris, ncams, res[0], res[1], int(self.prim is not None))
        if self._ws is None or self._ws.numel() < need:
            self._ws = None
            self._ws = torch.empty(need, dtype=torch.uint8, device=self.device)
        return self._ws

    def batch_size(self, res) -> int:
        per = _lib.size("fpvs_gt_pvs_workspace_size", self.ntris, 1, res[0], res[1], int(self.prim is not None))
        return max(1, int(WORKSPACE_BUDGET // max(per, 1)))

    def run(self, cams, frustum, dims, resolution, depth_mode: str = "linear", out=None, geometry=None):
        """GT bits (uint8 CUDA tensor, padded to 4 bytes) for camera list ``cams``."""
        torch = _torch()
        nx, ny, nz = (int(v) for v in dims)
        if nx % 8:
            raise ValueError(f"N_x must be divisible by 8, got {nx}")
        nbytes = nx * ny * nz // 8
        padded = (nbytes + 3) & ~3
        if out is None:
            out = torch.zeros(padded, dtype=torch.uint8, device=self.device)
        rows = _cam_rows(cams)
        fr = Frustum.of(frustum).c_struct()
        res = (int(resolution[0]), int(resolution[1]))
        if len(rows) == 0:
            out.zero_()
            return out[:nbytes]
        geo = geometry
        if geometry is not None and (geometry.numel() != padded or geometry.data_ptr() % 4):
            geo = torch.zeros(padded, dtype=torch.uint8, device=self.device)
            geo[:nbytes].copy_(geometry[:nbytes])
        bs = min(len(rows), self.batch_size(res))
        for i in range(0, len(rows), bs):
            part = torch.from_numpy(np.ascontiguousarray(rows[i:i + bs])).to(self.device)
            ws = self._ws_for(len(part), res)
            _lib.call("fpvs_gt_pvs", _lib.ptr(self.verts), self.verts.shape[0], _lib.ptr(self.tris), self.ntris,
                      _lib.ptr(self.prim), _lib.ptr(part), len(part), res[0], res[1], ctypes.byref(fr), nx, ny, nz,
                      0 if depth_mode == "linear" else 1, int(i > 0), _lib.ptr(out), _lib.ptr(geo), _lib.ptr(ws),
                      ws.numel(), _lib.stream_ptr())
        if geo is not None and geo is not geometry:
            geometry[:nbytes].copy_(geo[:nbytes])
        return out[:nbytes]

    def for_cell(self, cell, dims, ocfg: OracleConfig | None = None, fcfg: FroxelizeConfig | None = None,
                 cameras=None, out=None, geometry=None):
        """oracle.py:141-172 for one viewcell: sample cameras, render, reproject."""
        ocfg = ocfg or OracleConfig()
        fcfg = fcfg or FroxelizeConfig()
        cams = cameras if cameras is not None else views.sample_viewpoints(cell, ocfg.viewpoints, ocfg.mode,
                                                                           ocfg.seed)
        res = ocfg.resolution_for(dims)
        return self.run(cams, views.build_viewcell_frustum(cell), dims, res, fcfg.depth_mode, out=out,
                        geometry=geometry)


def compute_gt_pvs(scene, cell, dims, ocfg: OracleConfig | None = None, fcfg: FroxelizeConfig | None = None,
                   geometry: FroxelGrid | None = None, cameras: list | None = None) -> FroxelGrid:
    """oracle.py:141-172 on the device: host scene in, host ``FroxelGrid`` (role gt_pvs) out."""
    torch = _torch()
    fcfg = fcfg or FroxelizeConfig()
    nx, ny, nz = (int(v) for v in dims)
    gt = FroxelGrid((nx, ny, nz), role="gt_pvs", supersample=fcfg.supersample)
    g = GtPvs(scene.vertices, scene.triangles, getattr(scene, "primitive_ids", None))
    geo = None if geometry is None else torch.from_numpy(geometry.bits.copy()).to(g.device)
    bits = g.for_cell(cell, gt.dims, ocfg, fcfg, cameras=cameras, geometry=geo)
    gt.bits[:] = bits.cpu().numpy()
    if geometry is not None:
        geometry.bits[:] = geo.cpu().numpy()
    return gt
