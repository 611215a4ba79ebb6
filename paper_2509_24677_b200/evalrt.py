"""The PVS consumption side on the device.

Drop-ins for pkg/src/froxelpvs/evalrt.py and froxel.py:397-417:

* ``froxel_metrics(pred, gt)`` — popcount TP/FP/FN/GTP and FNR/FPR
  (evalrt.py:38-59) via ``fpvs_bits_confusion``;
* ``froxel_id_map(scene, frustum, dims, cfg)`` — returns an ``IdMap``: the
  froxel -> primitive-id map of froxel.py:397-417 held as its scene +
  frustum on the device.  ``cull`` consumes it with ONE fused raster pass
  (``fpvs_froxel_cull``: every fragment reads the PVS bit of its
  froxel and marks its triangle) instead of iterating a dict; reading it as
  a mapping materialises the reference's dict from ``fpvs_froxel_pairs``;
* ``cull(scene, pvs, id_map)`` (evalrt.py:62-68);
* ``render_depth(scene, camera, resolution)`` (oracle.py:107-138) ->
  ``DepthBuffer`` via ``fpvs_render_depth``;
* ``pixel_error_rate`` (evalrt.py:71-84) and ``far_field_merge``
  (evalrt.py:87-106) on top of those.

There is no CPU path: every call raises without the CUDA library.
"""

from __future__ import annotations

import ctypes
from collections.abc import Mapping
from dataclasses import dataclass

import numpy as np

from . import _lib, views
from .froxel import FroxelGrid
from .froxelize import FroxelizeConfig, Froxelizer, Frustum


def _torch():
    import torch
    return torch


@dataclass
class MetricsRecord:
    """evalrt.py:21-35."""

    frame: int
    fnr: float
    fpr: float
    per: float
    tp: int
    fp: int
    fn: int
    gtp: int
    infer_ms: float = 0.0
    oracle_ms: float = 0.0
    gtp_zero: bool = False


def _padded_device_bits(bits, device="cuda"):
    torch = _torch()
    b = np.asarray(bits, dtype=np.uint8).reshape(-1)
    out = torch.zeros((b.size + 3) & ~3, dtype=torch.uint8, device=device)
    out[:b.size].copy_(torch.from_numpy(b))
    return out


def froxel_metrics(pred: FroxelGrid, gt: FroxelGrid, frame: int = 0, per: float = 0.0, infer_ms: float = 0.0,
                   oracle_ms: float = 0.0) -> MetricsRecord:
    """evalrt.py:38-59 with the counts from fpvs_bits_confusion."""
    torch = _torch()
    _lib.require_cuda()
    if tuple(pred.dims) != tuple(gt.dims):
        raise ValueError(f"grid dims mismatch: {pred.dims} vs {gt.dims}")
    p = torch.from_numpy(np.ascontiguousarray(pred.bits)).cuda()
    g = torch.from_numpy(np.ascontiguousarray(gt.bits)).cuda()
    ws = torch.empty(_lib.size("fpvs_bits_confusion_workspace_size", 1), dtype=torch.uint8, device="cuda")
    counts = torch.zeros(4, dtype=torch.int64, device="cuda")
    _lib.call("fpvs_bits_confusion", _lib.ptr(p), _lib.ptr(g), 1, p.numel(), _lib.ptr(counts), _lib.ptr(ws),
              ws.numel(), _lib.stream_ptr())
    tp, fp, fn, gtp = (int(v) for v in counts.cpu().tolist())
    if gtp == 0:
        return MetricsRecord(frame, 0.0, 0.0, per, tp, fp, fn, gtp, infer_ms, oracle_ms, gtp_zero=True)
    return MetricsRecord(frame, fn / gtp, fp / gtp, per, tp, fp, fn, gtp, infer_ms, oracle_ms)


def _prim_ids(scene, ntris):
    pids = getattr(scene, "primitive_ids", None)
    return np.arange(ntris, dtype=np.int64) if pids is None else np.asarray(pids, dtype=np.int64).reshape(-1)


class IdMap(Mapping):
    """froxel.py:397-417's froxel -> {primitive ids} map, kept as (scene, frustum)
    on the device.  ``cull`` uses it without materialising; iterating / indexing
    builds the reference's dict once (fpvs_froxel_pairs + a device unique)."""

    def __init__(self, scene, frustum, dims, cfg: FroxelizeConfig | None = None):
        self.cfg = cfg or FroxelizeConfig()
        nx, ny, nz = (int(d) for d in dims)
        if nx % 8 != 0:
            raise ValueError(f"N_x must be divisible by 8, got {nx}")
        self.dims = (nx, ny, nz)
        self.fz = Froxelizer(scene.vertices, scene.triangles)
        self.prim_ids = _prim_ids(scene, self.fz.ntris)
        self.frustum = Frustum.of(frustum)
        self._dict = None

    def _call(self, name, *args):
        nx, ny, nz = self.dims
        ws = self.fz.workspace(self.dims, self.cfg.supersample, self.cfg.mode)
        c = self.frustum.c_struct()
        if self.cfg.mode == "ortho":
            name += "_ortho"
        _lib.call(name, _lib.ptr(self.fz.verts), self.fz.verts.shape[0], _lib.ptr(self.fz.tris), self.fz.ntris,
                  ctypes.byref(c), nx, ny, nz, int(self.cfg.supersample),
                  0 if self.cfg.depth_mode == "linear" else 1, *args, _lib.ptr(ws), ws.numel(), _lib.stream_ptr())

    def kept_triangles(self, pvs_bits_device):
        """uint8 [T] device flags: triangle has a fragment in a PVS froxel."""
        torch = _torch()
        kept = torch.empty(max(self.fz.ntris, 1), dtype=torch.uint8, device=self.fz.device)
        self._call("fpvs_froxel_cull", _lib.ptr(pvs_bits_device), _lib.ptr(kept))
        return kept[:self.fz.ntris]

    def _materialise(self):
        if self._dict is not None:
            return self._dict
        torch = _torch()
        nx, ny, _ = self.dims
        mapping: dict = {}
        if self.fz.ntris:
            self.fz.run(self.frustum, self.dims, self.cfg)
            cap = max(self.fz.samples(), 1)
            pairs = torch.empty(cap, dtype=torch.int64, device=self.fz.device)
            n = torch.zeros(1, dtype=torch.int64, device=self.fz.device)
            self._call("fpvs_froxel_pairs", _lib.ptr(pairs), cap, _lib.ptr(n))
            keys = torch.unique(pairs[:min(int(n.item()), cap)]).cpu().numpy()
            flat, tri = keys // self.fz.ntris, keys % self.fz.ntris
            fp = np.unique(np.column_stack([flat, self.prim_ids[tri]]), axis=0)
            for f, pid in fp:
                coord = (int(f % nx), int((f // nx) % ny), int(f // (nx * ny)))
                mapping.setdefault(coord, set()).add(int(pid))
        self._dict = mapping
        return mapping

    def __getitem__(self, key):
        return self._materialise()[key]

    def __iter__(self):
        return iter(self._materialise())

    def __len__(self):
        return len(self._materialise())


def froxel_id_map(scene, frustum, dims, cfg: FroxelizeConfig | None = None) -> IdMap:
    """froxel.py:397-417 (perspective or ortho fragment stream) -> device-backed ``IdMap``."""
    return IdMap(scene, frustum, dims, cfg)


def cull(scene, pvs: FroxelGrid, id_map) -> set:
    """evalrt.py:62-68: primitive ids that appear in at least one PVS-marked froxel."""
    if not isinstance(id_map, IdMap):
        raise TypeError("cull() takes the IdMap returned by paper_2509_24677_b200.evalrt.froxel_id_map")
    if tuple(pvs.dims) != id_map.dims:
        raise ValueError(f"pvs dims {pvs.dims} do not match the id map's {id_map.dims}")
    kept = id_map.kept_triangles(_padded_device_bits(pvs.bits, id_map.fz.device)).cpu().numpy().astype(bool)
    return set(int(i) for i in np.unique(id_map.prim_ids[kept]))


@dataclass
class DepthBuffer:
    """oracle.py:48-62: depth (+inf empty) and prim (-1 empty), indexed [row, col]."""

    depth: np.ndarray
    prim: np.ndarray
    near: float
    far: float

    @property
    def resolution(self) -> tuple:
        return self.depth.shape[1], self.depth.shape[0]

    def coverage(self) -> float:
        return float(np.isfinite(self.depth).mean())


def render_depth_device(vertices, triangles, prim_ids, cams, resolution, want_depth=True):
    """(depth [M,H,W] float64 or None, prim [M,H,W] int64) CUDA tensors for camera list ``cams``."""
    torch = _torch()
    _lib.require_cuda()
    from .gtpvs import _cam_rows
    w, h = int(resolution[0]), int(resolution[1])
    v = torch.from_numpy(np.ascontiguousarray(np.asarray(vertices, dtype=np.float64).reshape(-1, 3))).cuda()
    t = torch.from_numpy(np.ascontiguousarray(np.asarray(triangles, dtype=np.int64).reshape(-1, 3))).cuda()
    p = torch.from_numpy(np.ascontiguousarray(np.asarray(prim_ids, dtype=np.int64).reshape(-1))).cuda()
    rows = torch.from_numpy(_cam_rows(cams)).cuda()
    m = rows.shape[0]
    depth = torch.empty((m, h, w), dtype=torch.float64, device="cuda") if want_depth else None
    prim = torch.empty((m, h, w), dtype=torch.int64, device="cuda")
    ws = torch.empty(_lib.size("fpvs_gt_pvs_workspace_size", t.shape[0], m, w, h, 1), dtype=torch.uint8,
                     device="cuda")
    _lib.call("fpvs_render_depth", _lib.ptr(v), v.shape[0], _lib.ptr(t), t.shape[0], _lib.ptr(p), _lib.ptr(rows), m,
              w, h, _lib.ptr(depth), _lib.ptr(prim), _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
    return depth, prim


def render_depth(scene, camera, resolution) -> DepthBuffer:
    """oracle.py:107-138 on the device."""
    cam = camera if isinstance(camera, views.Camera) else views.Camera.of(camera)
    t = np.asarray(scene.triangles, dtype=np.int64).reshape(-1, 3)
    depth, prim = render_depth_device(scene.vertices, t, _prim_ids(scene, len(t)), [cam], resolution)
    return DepthBuffer(depth[0].cpu().numpy(), prim[0].cpu().numpy(), cam.near, cam.far)


def _subset(scene, keep_ids):
    """core.py:163-167: triangles whose primitive id is kept."""
    t = np.asarray(scene.triangles, dtype=np.int64).reshape(-1, 3)
    pids = _prim_ids(scene, len(t))
    mask = np.isin(pids, np.asarray(sorted(set(int(i) for i in keep_ids)), dtype=np.int64))
    return scene.vertices, t[mask], pids[mask]


def pixel_error_rate(scene, camera, pvs: FroxelGrid, id_map, resolution=(256, 256)) -> float:
    """evalrt.py:71-84: fraction of pixels whose visible primitive changes after culling."""
    cam = camera if isinstance(camera, views.Camera) else views.Camera.of(camera)
    kept = cull(scene, pvs, id_map)
    t = np.asarray(scene.triangles, dtype=np.int64).reshape(-1, 3)
    _, full = render_depth_device(scene.vertices, t, _prim_ids(scene, len(t)), [cam], resolution, want_depth=False)
    v, ts, ps = _subset(scene, kept)
    _, culled = render_depth_device(v, ts, ps, [cam], resolution, want_depth=False)
    return float((full != culled).double().mean().item())


def far_field_merge(scene, cell, pvs: FroxelGrid, id_map, threshold_distance: float, resolution=(256, 256)) -> set:
    """evalrt.py:87-106: culled set plus every id whose nearest visible fragment,
    seen from the enlarged frustum's origin, lies beyond the threshold."""
    torch = _torch()
    c = views.ViewCell.of(cell)
    if not (c.near < threshold_distance < c.far):
        raise ValueError("threshold must lie within the cell's (near, far) range")
    fr = views.build_viewcell_frustum(c)
    # the eye of evalrt.py:98-99: the frustum's own origin / axes / fov / near / far
    eye = views.Camera(tuple(fr._o), tuple(fr._basis[2]), tuple(fr._basis[1]), tuple(fr._basis[0]),
                       c.fov_deg + 2 * c.beta_deg, fr.near, fr.far)
    t = np.asarray(scene.triangles, dtype=np.int64).reshape(-1, 3)
    depth, prim = render_depth_device(scene.vertices, t, _prim_ids(scene, len(t)), [eye], resolution)
    far_mask = (prim >= 0) & ((depth - c.displacement) > threshold_distance)
    far_ids = set(int(i) for i in torch.unique(prim[far_mask]).cpu().tolist())
    return cull(scene, pvs, id_map) | far_ids
