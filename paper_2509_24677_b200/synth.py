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
