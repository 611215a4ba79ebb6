"""numpy restatement of the reference's perspective froxelizer (test infrastructure).

TEST INFRASTRUCTURE ONLY: imported by tests/ and bench.py's CPU legs as the
checker / CPU baseline for ``fpvs_froxelize``; the product package never
imports it.

Follows pkg/src/froxelpvs/froxel.py, perspective mode:
* camera space ``(v - o) @ basis.T`` (froxel.py:288-289) — numpy's matmul,
  exactly as the reference evaluates it;
* frustum cull ``max z > near and min z < far``, triangles with ``min z <
  near`` clipped against ``z >= near`` by Sutherland-Hodgman and fanned as
  ``(p0, pk, pk+1)`` (froxel.py:203-219, 292-325);
* projection ``u = (0.5 + 0.5 x / (z h)) W`` and ``1/z`` per vertex
  (froxel.py:322-325);
* coverage at pixel centres with inclusive edge tests on the barycentrics of
  vertices 1 and 2 relative to vertex 0, bbox ``ceil(min-0.5) .. floor(max-0.5)``
  clipped to the screen, degenerate ``|den| <= 1e-12`` skipped
  (froxel.py:229-285);
* perspective-correct depth (linear or log) kept on ``0 <= w <= 1`` and
  quantized ``floor(uvw * dims)`` clamped (froxel.py:28-42, 328-348);
* bits packed LSB-first along x (froxel.py:115-118).

Unlike the reference (flat (triangle, sample) pair chunks over all
triangles) this walks one triangle's bounding box at a time; the arithmetic
per sample is the same expression sequence, so the grids are identical —
pinned against the reference's own output in tests/golden/froxelize.npz.
"""

from __future__ import annotations

import numpy as np

DEGEN_EPS = 1e-12


def _clip_near(poly, near):
    """Sutherland-Hodgman against z >= near (froxel.py:203-219)."""
    d = poly[:, 2] - near
    out = []
    for i in range(len(poly)):
        j = (i + 1) % len(poly)
        if d[i] >= 0:
            out.append(poly[i])
        if (d[i] >= 0) != (d[j] >= 0):
            t = d[i] / (d[i] - d[j])
            out.append(poly[i] + t * (poly[j] - poly[i]))
    return np.asarray(out, dtype=np.float64).reshape(-1, 3)


def camera_triangles(verts, tris, origin, basis, near, far, with_src=False):
    """Camera-space triangles after cull + near clip: (T', 3, 3) float64
    (and the source triangle of each when ``with_src``)."""
    verts = np.asarray(verts, dtype=np.float64).reshape(-1, 3)
    tris = np.asarray(tris, dtype=np.int64).reshape(-1, 3)
    if len(tris) == 0:
        return (np.zeros((0, 3, 3)), np.zeros(0, np.int64)) if with_src else np.zeros((0, 3, 3))
    cam = (verts - np.asarray(origin, dtype=np.float64)) @ np.asarray(basis, dtype=np.float64).T
    ct = cam[tris]
    z = ct[:, :, 2]
    cand = (z.max(axis=1) > near) & (z.min(axis=1) < far)
    clean = np.nonzero(cand & (z.min(axis=1) >= near))[0]
    keep, src = [ct[clean]], [clean]
    for t in np.nonzero(cand & (z.min(axis=1) < near))[0]:
        poly = _clip_near(ct[t], near)
        for k in range(1, len(poly) - 1):
            keep.append(poly[[0, k, k + 1]][None])
            src.append(np.array([t]))
    out = np.concatenate(keep, axis=0)
    return (out, np.concatenate(src)) if with_src else out


def froxelize(verts, tris, origin, basis, half_extent, near, far, dims, supersample=4, depth_mode="linear"):
    """Packed geometry grid (uint8, Nx*Ny*Nz/8) of the triangle scene."""
    nx, ny, nz = (int(v) for v in dims)
    if nx % 8:
        raise ValueError(f"N_x must be divisible by 8, got {nx}")
    bits = np.zeros(nx * ny * nz // 8, dtype=np.uint8)
    sx, sy = supersample * nx, supersample * ny
    cam = camera_triangles(verts, tris, origin, basis, near, far)
    if len(cam) == 0:
        return bits
    zc = cam[:, :, 2]
    scr_u = (0.5 + 0.5 * cam[:, :, 0] / (zc * half_extent)) * sx
    scr_v = (0.5 + 0.5 * cam[:, :, 1] / (zc * half_extent)) * sy
    invz = 1.0 / zc
    if depth_mode == "linear":
        wv = (1.0 / invz - near) / (far - near)
    else:
        wv = np.log(1.0 / (invz * near)) / np.log(far / near)
    d = np.array([nx, ny, nz], dtype=np.int64)
    row = nx // 8
    for t in range(len(cam)):
        u, v = scr_u[t], scr_v[t]
        e1x, e1y = u[1] - u[0], v[1] - v[0]
        e2x, e2y = u[2] - u[0], v[2] - v[0]
        den = e1x * e2y - e2x * e1y
        x0 = int(np.clip(np.ceil(u.min() - 0.5), 0, sx))
        x1 = int(np.clip(np.floor(u.max() - 0.5) + 1, 0, sx))
        y0 = int(np.clip(np.ceil(v.min() - 0.5), 0, sy))
        y1 = int(np.clip(np.floor(v.max() - 0.5) + 1, 0, sy))
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
        px, py, b1, b2 = px[m], py[m], b1[m], b2[m]
        iz = invz[t]
        inv = iz[0] + b1 * (iz[1] - iz[0]) + b2 * (iz[2] - iz[0])
        c1 = b1 * iz[1] / inv
        c2 = b2 * iz[2] / inv
        w = wv[t, 0] + c1 * (wv[t, 1] - wv[t, 0]) + c2 * (wv[t, 2] - wv[t, 0])
        k = (w >= 0) & (w <= 1)
        if not k.any():
            continue
        uvw = np.column_stack([(px[k] + 0.5) / sx, (py[k] + 0.5) / sy, w[k]])
        idx = np.clip(np.floor(uvw * d).astype(np.int64), 0, d - 1)
        byte = (idx[:, 0] >> 3) + row * (idx[:, 1] + ny * idx[:, 2])
        np.bitwise_or.at(bits, byte, (np.uint8(1) << (idx[:, 0] & 7).astype(np.uint8)).astype(np.uint8))
    return bits


# ---------------------------------------------------------------------------
# orthographic three-view mode (froxel.py:351-376)
# ---------------------------------------------------------------------------


def world_aabb(origin, basis, half_extent, near, far):
    """core.py:349-354 (unproject_ndc of the 8 NDC corners, linear depth)."""
    uvw = np.array([[u, v, w] for u in (0, 1) for v in (0, 1) for w in (0, 1)], dtype=np.float64)
    z = near + uvw[:, 2] * (far - near)
    x = (2.0 * uvw[:, 0] - 1.0) * half_extent * z
    y = (2.0 * uvw[:, 1] - 1.0) * half_extent * z
    corners = np.asarray(origin, dtype=np.float64) + np.column_stack([x, y, z]) @ np.asarray(basis, dtype=np.float64)
    return corners.min(axis=0), corners.max(axis=0)


def project_points(origin, basis, half_extent, near, far, pts, depth_mode="linear"):
    """core.py:380-405: (uvw, inside)."""
    local = (pts - np.asarray(origin, dtype=np.float64)) @ np.asarray(basis, dtype=np.float64).T
    x, y, z = local[:, 0], local[:, 1], local[:, 2]
    ahead = z > 0
    zs = np.where(ahead, z, 1.0)
    u = 0.5 + 0.5 * x / (zs * half_extent)
    v = 0.5 + 0.5 * y / (zs * half_extent)
    if depth_mode == "linear":
        w = (z - near) / (far - near)
    else:
        import math
        w = np.log(np.where(ahead, z, near) / near) / math.log(far / near)
    inside = ahead & (u >= 0) & (u <= 1) & (v >= 0) & (v <= 1) & (w >= 0) & (w <= 1)
    return np.column_stack([u, v, w]), inside


def froxelize_ortho(verts, tris, origin, basis, half_extent, near, far, dims, supersample=4, depth_mode="linear"):
    """Three axis-aligned orthographic passes over the frustum's world AABB, every
    covered sample point reprojected into the frustum (froxel.py:351-376)."""
    nx, ny, nz = (int(v) for v in dims)
    bits = np.zeros(nx * ny * nz // 8, dtype=np.uint8)
    verts = np.asarray(verts, dtype=np.float64).reshape(-1, 3)
    tris = np.asarray(tris, dtype=np.int64).reshape(-1, 3)
    if len(tris) == 0:
        return bits
    lo, hi = world_aabb(origin, basis, half_extent, near, far)
    extent = hi - lo
    spacing = extent.max() / (supersample * max(nx, ny, nz))
    counts = np.maximum(np.ceil(extent / spacing).astype(np.int64), 1)
    tv = verts[tris]
    live = np.nonzero(((tv.max(axis=1) >= lo) & (tv.min(axis=1) <= hi)).all(axis=1))[0]
    d = np.array([nx, ny, nz], dtype=np.int64)
    for a0, a1, ar in ((1, 2, 0), (2, 0, 1), (0, 1, 2)):
        t2 = (tv[live][:, :, [a0, a1]] - lo[[a0, a1]]) / spacing
        attrs = tv[live][:, :, ar]
        W, H = int(counts[a0]), int(counts[a1])
        for t in range(len(live)):
            u, v = t2[t, :, 0], t2[t, :, 1]
            e1x, e1y = u[1] - u[0], v[1] - v[0]
            e2x, e2y = u[2] - u[0], v[2] - v[0]
            den = e1x * e2y - e2x * e1y
            x0 = int(np.clip(np.ceil(u.min() - 0.5), 0, W))
            x1 = int(np.clip(np.floor(u.max() - 0.5) + 1, 0, W))
            y0 = int(np.clip(np.ceil(v.min() - 0.5), 0, H))
            y1 = int(np.clip(np.floor(v.max() - 0.5) + 1, 0, H))
            if not (abs(den) > DEGEN_EPS) or x1 <= x0 or y1 <= y0:
                continue
            sv, su = np.mgrid[y0:y1, x0:x1]
            su, sv = su.ravel(), sv.ravel()
            dx = (su + 0.5) - u[0]
            dy = (sv + 0.5) - v[0]
            b1 = (dx * e2y - e2x * dy) / den
            b2 = (e1x * dy - dx * e1y) / den
            b0 = 1.0 - b1 - b2
            m = (b0 >= 0) & (b1 >= 0) & (b2 >= 0)
            if not m.any():
                continue
            a = attrs[t]
            world = np.empty((int(m.sum()), 3))
            world[:, a0] = lo[a0] + (su[m] + 0.5) * spacing
            world[:, a1] = lo[a1] + (sv[m] + 0.5) * spacing
            world[:, ar] = a[0] + b1[m] * (a[1] - a[0]) + b2[m] * (a[2] - a[0])
            uvw, inside = project_points(origin, basis, half_extent, near, far, world, depth_mode)
            if not inside.any():
                continue
            idx = np.clip(np.floor(uvw[inside] * d).astype(np.int64), 0, d - 1)
            byte = (idx[:, 0] >> 3) + (nx // 8) * (idx[:, 1] + ny * idx[:, 2])
            np.bitwise_or.at(bits, byte, (np.uint8(1) << (idx[:, 0] & 7).astype(np.uint8)).astype(np.uint8))
    return bits
