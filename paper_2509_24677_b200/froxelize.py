"""Device froxelization: triangle scene -> packed geometry grid.

Drop-in for ``froxelpvs.froxel.froxelize`` (pkg/src/froxelpvs/froxel.py:387-394)
in both modes (``"perspective"``, froxel.py:328-348, and the three-view
``"ortho"``, froxel.py:351-376, via ``fpvs_froxelize_ortho``): same arguments (a scene with ``vertices`` /
``triangles``, a frustum with ``_o`` / ``_basis`` / ``half_extent`` / ``near`` /
``far``, dims, a ``FroxelizeConfig``), same ``FroxelGrid`` result, bit-for-bit
in both depth modes.  The work runs in ``fpvs_froxelize`` (csrc/froxelize.cu);
there is no CPU path — without the CUDA library the call raises.

``Froxelizer`` keeps the scene and workspace resident on the device for
repeated frusta (one viewcell after another over the same scene), writing
straight into a device packed-bit buffer that the PVS pipeline consumes
(``FramePipeline.in_bits``) with no host round trip.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .froxel import FroxelGrid


def _torch():
    import torch
    return torch


@dataclass
class FroxelizeConfig:
    """Mirror of froxel.py:45-61 (``supersample``, ``mode``, ``depth_mode``)."""

    supersample: int = 4
    mode: str = "perspective"
    depth_mode: str = "linear"

    def __post_init__(self):
        if self.supersample < 1:
            raise ValueError("supersample factor must be >= 1")
        if self.mode not in ("perspective", "ortho"):
            raise ValueError(f"unknown froxelize mode {self.mode!r}")
        if self.depth_mode not in ("linear", "log"):
            raise ValueError(f"unknown depth mode {self.depth_mode!r}")


class Frustum:
    """The rasterizer's view of core.py:297-325: origin, basis rows (right, up,
    forward), half extent tan(fov/2), near, far.  ``from_vectors`` normalises
    the axes exactly as Vec3.normalized does (core.py:61-68)."""

    def __init__(self, origin, basis, half_extent: float, near: float, far: float):
        self._o = np.asarray(origin, dtype=np.float64).reshape(3)
        self._basis = np.asarray(basis, dtype=np.float64).reshape(3, 3)
        self.half_extent = float(half_extent)
        self.near, self.far = float(near), float(far)
        if not (0.0 < self.near < self.far):
            raise ValueError("need 0 < near < far")

    @staticmethod
    def _unit(v):
        x, y, z = (float(c) for c in v)
        n = math.sqrt(x * x + y * y + z * z)
        if n == 0.0:
            raise ValueError("cannot normalize a zero vector")
        s = 1.0 / n
        return [x * s, y * s, z * s]

    @classmethod
    def from_vectors(cls, origin, forward, up, right, fov_deg: float, near: float, far: float) -> "Frustum":
        if not (0.0 < fov_deg < 180.0):
            raise ValueError(f"frustum fov must lie in (0, 180), got {fov_deg}")
        basis = [cls._unit(right), cls._unit(up), cls._unit(forward)]
        return cls(origin, basis, math.tan(math.radians(float(fov_deg)) / 2.0), near, far)

    @classmethod
    def of(cls, frustum) -> "Frustum":
        """Accept this class or the reference's Frustum (duck-typed)."""
        if isinstance(frustum, cls):
            return frustum
        return cls(frustum._o, frustum._basis, frustum.half_extent, frustum.near, frustum.far)

    def c_struct(self):
        fr = _lib.Frustum()
        for i in range(3):
            fr.origin[i] = float(self._o[i])
        for i, v in enumerate(self._basis.reshape(-1)):
            fr.basis[i] = float(v)
        fr.half_extent, fr.near_z, fr.far_z = self.half_extent, self.near, self.far
        return fr


def _check_dims(dims):
    nx, ny, nz = (int(v) for v in dims)
    if nx % 8 != 0:
        raise ValueError(f"N_x must be divisible by 8, got {nx}")
    if min(nx, ny, nz) <= 0:
        raise ValueError("grid dims must be positive")
    return nx, ny, nz


class Froxelizer:
    """A scene resident on the device, froxelized for any number of frusta.

    ``vertices`` float64 (V, 3), ``triangles`` int (T, 3) — host arrays or
    CUDA tensors.  ``run`` is stream-ordered and graph-capturable (no host
    sync, no allocation after the first call for a given dims)."""

    def __init__(self, vertices, triangles, device="cuda"):
        torch = _torch()
        _lib.require_cuda()
        self.verts = torch.as_tensor(np.asarray(vertices, dtype=np.float64).reshape(-1, 3)
                                     if not torch.is_tensor(vertices) else vertices,
                                     dtype=torch.float64, device=device).contiguous()
        tris = triangles if torch.is_tensor(triangles) else np.asarray(triangles, dtype=np.int64).reshape(-1, 3)
        self.tris = torch.as_tensor(tris, dtype=torch.int64, device=device).contiguous()
        if self.tris.numel() and not torch.is_tensor(triangles):
            t = np.asarray(triangles)
            if t.min() < 0 or t.max() >= self.verts.shape[0]:
                raise ValueError("triangle index out of range")
        self.device = device
        self._ws = None

    @property
    def ntris(self) -> int:
        return int(self.tris.shape[0])

    def workspace(self, dims, supersample: int, mode: str = "perspective"):
        torch = _torch()
        nx, ny, nz = dims
        fn = "fpvs_froxelize_ortho_workspace_size" if mode == "ortho" else "fpvs_froxelize_workspace_size"
        need = _lib.size(fn, self.ntris, nx, ny, nz, int(supersample))
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.empty(need, dtype=torch.uint8, device=self.device)
        return self._ws

    def run(self, frustum, dims, cfg: FroxelizeConfig | None = None, out=None):
        """Packed grid (uint8 CUDA tensor, Nx*Ny*Nz/8) of this scene in ``frustum``."""
        torch = _torch()
        cfg = cfg or FroxelizeConfig()
        nx, ny, nz = _check_dims(dims)
        fr = Frustum.of(frustum)
        nbytes = nx * ny * nz // 8
        if out is None:
            out = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        elif out.numel() != nbytes or out.dtype != torch.uint8:
            raise ValueError("output buffer does not match dims")
        ws = self.workspace((nx, ny, nz), cfg.supersample, cfg.mode)
        c = fr.c_struct()
        import ctypes
        _lib.call("fpvs_froxelize_ortho" if cfg.mode == "ortho" else "fpvs_froxelize", _lib.ptr(self.verts), self.verts.shape[0], _lib.ptr(self.tris), self.ntris,
                  ctypes.byref(c), nx, ny, nz, int(cfg.supersample), 0 if cfg.depth_mode == "linear" else 1,
                  _lib.ptr(out), _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
        return out

    def samples(self) -> int:
        """Candidate samples (sum of clipped screen bounding boxes) of the last run; syncs."""
        return int(_lib.load().fpvs_froxelize_samples(_lib.ptr(self._ws), _lib.stream_ptr()))


def froxelize(scene, frustum, dims, cfg: FroxelizeConfig | None = None) -> FroxelGrid:
    """froxel.py:387-394 on the device: host scene in, host ``FroxelGrid`` out."""
    cfg = cfg or FroxelizeConfig()
    nx, ny, nz = _check_dims(dims)
    fz = Froxelizer(scene.vertices, scene.triangles)
    bits = fz.run(frustum, (nx, ny, nz), cfg)
    return FroxelGrid((nx, ny, nz), role="geometry", supersample=cfg.supersample, bits=bits.cpu().numpy())
