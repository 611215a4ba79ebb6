"""numpy restatement of the reference's GT-PVS generator (test infrastructure).

TEST INFRASTRUCTURE ONLY: imported by tests/ and bench.py's CPU legs as the
checker / CPU baseline for ``fpvs_gt_pvs``; the product package never
imports it.

Follows pkg/src/froxelpvs/oracle.py:107-172 (``render_depth``,
``compute_gt_pvs``) and core.py:380-452 (``project_points``,
``unproject_pixels``):
* per camera, the scene is culled / near-clipped / projected like the
  froxelizer (froxel.py:292-325) at the depth-buffer resolution, every
  covered pixel centre gets depth ``1 / interp(1/z)`` kept when ``<= far``,
  the z-test keeps the minimum, exact ties resolve to the smallest primitive
  id, and pixels whose winning id is ``>= 0`` are the fragments
  (oracle.py:107-138);
* each fragment is unprojected from its camera (``x = (2 (px+0.5)/W - 1) h z``),
  projected into the viewcell frustum and, when inside, quantized and OR-ed
  into the GT grid — and into ``geometry`` when given (oracle.py:141-172).
Per-triangle bounding-box walks replace the reference's flat pair chunks;
the per-sample expressions are the same, so the grids are identical —
pinned against the reference's own output in tests/golden/gtpvs.npz.
"""

from __future__ import annotations

import math

import numpy as np

from .froxelize import DEGEN_EPS, camera_triangles


def render_depth(verts, tris, prim_ids, cam, width, height):
    """(depth (H, W) float64 with +inf where empty, prim (H, W) int64 with -1)."""
    origin, basis, he, near, far = cam
    zflat = np.full(width * height, np.inf)
    iflat = np.full(width * height, np.iinfo(np.int64).max, dtype=np.int64)
    ct, src = camera_triangles(verts, tris, origin, basis, near, far, with_src=True)
    frags = []
    if len(ct):
        zc = ct[:, :, 2]
        su = (0.5 + 0.5 * ct[:, :, 0] / (zc * he)) * width
        sv = (0.5 + 0.5 * ct[:, :, 1] / (zc * he)) * height
        invz = 1.0 / zc
        for t in range(len(ct)):
            u, v, iz = su[t], sv[t], invz[t]
            e1x, e1y = u[1] - u[0], v[1] - v[0]
            e2x, e2y = u[2] - u[0], v[2] - v[0]
            den = e1x * e2y - e2x * e1y
            x0 = int(np.clip(np.ceil(u.min() - 0.5), 0, width))
            x1 = int(np.clip(np.floor(u.max() - 0.5) + 1, 0, width))
            y0 = int(np.clip(np.ceil(v.min() - 0.5), 0, height))
            y1 = int(np.clip(np.floor(v.max() - 0.5) + 1, 0, height))
            if not (abs(den) > DEGEN_EPS) or x1 <= x0 or y1 <= y0:
                continue
            py, px = np.mgrid[y0:y1, x0:x1]
            px, py = px.ravel(), py.ravel()
            dx = (px + 0.5) - u[0]
            dy = (py + 0.5) - v[0]
            b1 = (dx * e2y - e2x * dy) / den
            b2 = (e1x * dy - dx * e1y) / den
            b0 = 1.0 - b1 - b2
            m = (b0 >= 0) & (b1 >= 0) & (b2 >= 0)
            if not m.any():
                continue
            depth = 1.0 / (iz[0] + b1[m] * (iz[1] - iz[0]) + b2[m] * (iz[2] - iz[0]))
            k = depth <= far
            if not k.any():
                continue
            flat = py[m][k] * width + px[m][k]
            np.minimum.at(zflat, flat, depth[k])
            frags.append((flat, depth[k], np.full(int(k.sum()), prim_ids[src[t]], dtype=np.int64)))
    for flat, depth, pid in frags:
        win = depth <= zflat[flat]
        np.minimum.at(iflat, flat[win], pid[win])
    prim = np.where(np.isfinite(zflat), iflat, -1).reshape(height, width)
    return zflat.reshape(height, width), prim


def reproject(cam, frustum, px, py, depth, width, height, depth_mode="linear"):
    """core.py:433-452 then core.py:380-405: (uvw, inside)."""
    origin, basis, he, _near, _far = cam
    px = np.asarray(px, dtype=np.float64)
    py = np.asarray(py, dtype=np.float64)
    z = np.asarray(depth, dtype=np.float64)
    x = (2.0 * (px + 0.5) / width - 1.0) * he * z
    y = (2.0 * (py + 0.5) / height - 1.0) * he * z
    world = np.asarray(origin, dtype=np.float64) + np.column_stack([x, y, z]) @ np.asarray(basis, dtype=np.float64)
    fo, fb, fh, fn, ff = frustum
    local = (world - np.asarray(fo, dtype=np.float64)) @ np.asarray(fb, dtype=np.float64).T
    lx, ly, lz = local[:, 0], local[:, 1], local[:, 2]
    ahead = lz > 0
    zs = np.where(ahead, lz, 1.0)
    u = 0.5 + 0.5 * lx / (zs * fh)
    v = 0.5 + 0.5 * ly / (zs * fh)
    if depth_mode == "linear":
        w = (lz - fn) / (ff - fn)
    else:
        w = np.log(np.where(ahead, lz, fn) / fn) / math.log(ff / fn)
    inside = ahead & (u >= 0) & (u <= 1) & (v >= 0) & (v <= 1) & (w >= 0) & (w <= 1)
    return np.column_stack([u, v, w]), inside


def gt_pvs(verts, tris, cams, frustum, dims, resolution, depth_mode="linear", prim_ids=None, geometry=None):
    """Packed GT PVS grid (uint8) over the cameras; ORs into ``geometry`` (packed, in place) too."""
    nx, ny, nz = (int(v) for v in dims)
    w, h = (int(v) for v in resolution)
    tris = np.asarray(tris, dtype=np.int64).reshape(-1, 3)
    pids = np.arange(len(tris), dtype=np.int64) if prim_ids is None else np.asarray(prim_ids, dtype=np.int64)
    bits = np.zeros(nx * ny * nz // 8, dtype=np.uint8)
    d = np.array([nx, ny, nz], dtype=np.int64)
    for cam in cams:
        depth, prim = render_depth(verts, tris, pids, cam, w, h)
        rows, cols = np.nonzero(prim >= 0)
        if len(rows) == 0:
            continue
        uvw, inside = reproject(cam, frustum, cols, rows, depth[rows, cols], w, h, depth_mode)
        if not inside.any():
            continue
        idx = np.clip(np.floor(uvw[inside] * d).astype(np.int64), 0, d - 1)
        byte = (idx[:, 0] >> 3) + (nx // 8) * (idx[:, 1] + ny * idx[:, 2])
        mask = (np.uint8(1) << (idx[:, 0] & 7).astype(np.uint8)).astype(np.uint8)
        np.bitwise_or.at(bits, byte, mask)
        if geometry is not None:
            np.bitwise_or.at(geometry, byte, mask)
    return bits
