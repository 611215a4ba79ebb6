"""Seeded synthetic froxel grids and PVS labels (BASELINE.json configs 1-5).

The paper's scenes (Viking Village, Robot Lab, Sponza, City) are
not available, so seeded axis-aligned box stampings stand in for them.  These
are *input synthesis* rules pinned by this repo, not part of
the reference:

* ``box_grid(dims, n, lo, hi, seed)``: ``rng = np.random.default_rng(seed)``;
  edges ``E = rng.integers(lo, hi+1, size=(n, 3))`` then positions
  ``P = rng.integers(0, dims, size=(n, 3))``; box ``[P, P+E)`` is stamped with
  ones, clipped at the border.
* ``box_grid_density(dims, target, lo, hi, seed)``: the same rule over a pool
  of ``n_pool`` boxes; the stamped prefix length is bisected so that the
  occupancy is the smallest prefix reaching ``target``.
* ``first_hit_labels(occ, radius=2)`` (row LBL): with
  ``zf(x, y) = min{z : occ(x, y, z)}``, a froxel is visible iff it is occupied
  and ``z == zf(x+dx, y+dy)`` for some ``|dx|, |dy| <= radius``.  This keeps
  V ⊆ G as PAPER.md:203 requires.

Grids are (Nx, Ny, Nz) with z the depth axis, as in the reference.
"""

from __future__ import annotations

import numpy as np


def _stamp(dims, lo_corner, hi_corner) -> np.ndarray:
    """Union of boxes [lo, hi) via a 3-D difference array (exact, O(N + n))."""
    nx, ny, nz = dims
    acc = np.zeros((nx + 1, ny + 1, nz + 1), np.int32)
    lo = np.asarray(lo_corner, np.int64)
    hi = np.minimum(np.asarray(hi_corner, np.int64), np.array(dims))
    for sx, ix in ((1, lo[:, 0]), (-1, hi[:, 0])):
        for sy, iy in ((1, lo[:, 1]), (-1, hi[:, 1])):
            for sz, iz in ((1, lo[:, 2]), (-1, hi[:, 2])):
                np.add.at(acc, (ix, iy, iz), sx * sy * sz)
    occ = acc.cumsum(0).cumsum(1).cumsum(2)[:nx, :ny, :nz]
    return occ > 0


def box_grid(dims, n_boxes: int, lo: int, hi: int, seed: int) -> np.ndarray:
    """Bool (Nx, Ny, Nz) occupancy from ``n_boxes`` seeded boxes."""
    rng = np.random.default_rng(seed)
    e = rng.integers(lo, hi + 1, size=(n_boxes, 3))
    p = rng.integers(0, np.asarray(dims), size=(n_boxes, 3))
    return _stamp(dims, p, p + e)


def box_grid_density(dims, target: float, lo: int, hi: int, seed: int,
                     n_pool: int | None = None):
    """(occupancy, n_boxes): smallest seeded prefix whose density >= target."""
    vol = float(np.prod(dims))
    mean_vol = ((lo + hi) / 2.0) ** 3
    if n_pool is None:
        n_pool = int(max(64, 8 * target * vol / mean_vol))
    rng = np.random.default_rng(seed)
    e = rng.integers(lo, hi + 1, size=(n_pool, 3))
    p = rng.integers(0, np.asarray(dims), size=(n_pool, 3))
    a, b = 1, n_pool
    while a < b:
        m = (a + b) // 2
        if _stamp(dims, p[:m], p[:m] + e[:m]).mean() >= target:
            b = m
        else:
            a = m + 1
    return _stamp(dims, p[:a], p[:a] + e[:a]), a


def first_hit_labels(occ: np.ndarray, radius: int = 2) -> np.ndarray:
    """Synthetic PVS labels (row LBL): occupied and first hit of a nearby column."""
    occ = np.asarray(occ, bool)
    nx, ny, nz = occ.shape
    big = np.int64(nz)
    zf = np.where(occ.any(axis=2), occ.argmax(axis=2), big)       # (Nx, Ny)
    zpad = np.full((nx + 2 * radius, ny + 2 * radius), big, np.int64)
    zpad[radius:radius + nx, radius:radius + ny] = zf
    z = np.arange(nz)[None, None, :]
    vis = np.zeros_like(occ)
    for dx in range(-radius, radius + 1):
        for dy in range(-radius, radius + 1):
            zn = zpad[radius + dx:radius + dx + nx, radius + dy:radius + dy + ny]
            vis |= z == zn[:, :, None]
    return vis & occ


def first_hit_labels_bits(bits, B: int, grid_dims, radius: int = 2, out=None, stream=None):
    """The same labels on the device from packed geometry bits (fpvs_first_hit_labels):
    B packed (Nx, Ny, Nz) grids in, B packed label grids out (CUDA uint8)."""
    import torch

    from . import _lib
    nx, ny, nz = grid_dims
    if out is None:
        out = torch.empty(B * nx * ny * nz // 8, dtype=torch.uint8, device=bits.device)
    ws = torch.empty(B * nx * ny, dtype=torch.int32, device=bits.device)
    _lib.call("fpvs_first_hit_labels", _lib.ptr(bits), B, nx, ny, nz, int(radius), _lib.ptr(out), _lib.ptr(ws),
              _lib.stream_ptr(stream))
    return out


# BASELINE.json config shapes ------------------------------------------------

def config1_grid(seed: int = 0) -> np.ndarray:
    return box_grid((64, 64, 32), 200, 1, 6, seed)


def config2_grid(seed: int = 1) -> np.ndarray:
    return box_grid((256, 256, 256), 4000, 1, 12, seed)


def config3_grid(i: int):
    """Grid i of the 64-grid batch: seed 100+i, target density U(1%, 6%)."""
    seed = 100 + i
    target = float(np.random.default_rng(seed).uniform(0.01, 0.06))
    occ, _ = box_grid_density((64, 64, 32), target, 1, 6, seed + 1_000_000)
    return occ


def config4_grid(density: float, seed: int = 4) -> np.ndarray:
    occ, _ = box_grid_density((256, 256, 256), density, 1, 12, seed)
    return occ


def config5_pair(rank: int, i: int):
    """(geometry, labels) for grid i of rank ``rank``: 128^3 at ~4% density."""
    seed = 5000 + 64 * rank + i
    occ, _ = box_grid_density((128, 128, 128), 0.04, 1, 8, seed)
    return occ, first_hit_labels(occ)


# --------------------------------------------------------------- triangle scenes
def _uv_sphere(nu: int, nv: int):
    """Closed lat-long sphere mesh of radius 1: (verts, tris)."""
    th = np.linspace(0, np.pi, nv + 1)[1:-1]
    ph = np.linspace(0, 2 * np.pi, nu, endpoint=False)
    ring = np.stack([np.sin(th)[:, None] * np.cos(ph)[None], np.cos(th)[:, None] + 0 * ph[None],
                     np.sin(th)[:, None] * np.sin(ph)[None]], axis=-1).reshape(-1, 3)
    verts = np.concatenate([[[0, 1, 0]], ring, [[0, -1, 0]]])
    tris = []
    for j in range(nu):
        tris.append([0, 1 + (j + 1) % nu, 1 + j])
    for i in range(nv - 2):
        a, b = 1 + i * nu, 1 + (i + 1) * nu
        for j in range(nu):
            k = (j + 1) % nu
            tris += [[a + j, a + k, b + j], [a + k, b + k, b + j]]
    last, pole = 1 + (nv - 2) * nu, len(verts) - 1
    for j in range(nu):
        tris.append([last + j, last + (j + 1) % nu, pole])
    return verts.astype(np.float64), np.asarray(tris, dtype=np.int64)


def _grid_quad(n: int):
    """Unit quad [-1,1]^2 in the xz plane tessellated into 2 n^2 triangles."""
    t = np.linspace(-1, 1, n + 1)
    x, z = np.meshgrid(t, t, indexing="ij")
    verts = np.stack([x.ravel(), 0 * x.ravel(), z.ravel()], axis=1)
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    a = (i * (n + 1) + j).ravel()
    tris = np.concatenate([np.stack([a, a + 1, a + n + 2], 1), np.stack([a, a + n + 2, a + n + 1], 1)])
    return verts, tris.astype(np.int64)


def _rot(rng):
    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    w, x, y, z = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
                     [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
                     [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]])


def froxel_scene(seed: int = 0, n_objects: int = 12, detail: int = 12, extent: float = 12.0):
    """Seeded triangle scene of the reference generator's kind (scenegen.py:312-372):
    a floor and a back wall spanning the view plus ``n_objects`` rotated,
    anisotropically scaled closed meshes around a viewcell at the origin.
    Returns (vertices float64 (V,3), triangles int64 (T,3), frustum args) where
    the frustum args are (origin, forward, up, right, fov_deg, near, far) of a
    viewcell frustum (core.py:361-373) looking along a random yaw."""
    rng = np.random.Generator(np.random.PCG64(seed))
    vs, ts, n = [], [], 0

    def add(v, t):
        nonlocal n
        vs.append(v)
        ts.append(t + n)
        n += len(v)

    sv, st = _uv_sphere(detail, max(3, detail // 2))
    cv = np.array([[x, y, z] for x in (-1, 1) for y in (-1, 1) for z in (-1, 1)], dtype=np.float64)
    ct = np.array([[0, 1, 3], [0, 3, 2], [4, 6, 7], [4, 7, 5], [0, 4, 5], [0, 5, 1],
                   [2, 3, 7], [2, 7, 6], [0, 2, 6], [0, 6, 4], [1, 5, 7], [1, 7, 3]], dtype=np.int64)
    for _ in range(n_objects):
        v, t = (sv, st) if rng.random() < 0.5 else (cv, ct)
        scale = np.exp(rng.uniform(np.log(0.5), np.log(4.0), size=3))
        pos = np.array([rng.uniform(-extent, extent), rng.uniform(0.2, 4.0), rng.uniform(-extent, extent)])
        add((v * scale) @ _rot(rng).T + pos, t)
    gq, gt = _grid_quad(max(1, detail // 2))
    span = 2.5 * extent
    add(gq * span, gt)                                                  # floor (y = 0)
    yaw = rng.uniform(0, 2 * np.pi)
    fwd = np.array([np.sin(yaw), 0.0, np.cos(yaw)])
    right = np.array([fwd[2], 0.0, -fwd[0]])
    wall = gq[:, [0, 2, 1]] * span                                      # xy plane
    wall = wall[:, 0:1] * right + wall[:, 1:2] * np.array([0.0, 1.0, 0.0]) + 1.5 * extent * fwd
    add(wall, gt)
    verts, tris = np.concatenate(vs), np.concatenate(ts)
    height = rng.uniform(0.8, 2.2)
    radius, fov, beta, near, far = 0.3, 60.0, 15.0, 0.3, 20.0
    h = np.tan(np.radians(fov) / 2)
    disp = radius / h
    origin = np.array([0.0, height, 0.0]) - disp * fwd
    up = np.array([0.0, 1.0, 0.0])
    return verts, tris, (origin, fwd, up, -right, fov + 2 * beta, disp, disp + far)
