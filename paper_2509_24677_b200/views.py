"""Viewcells, cameras and viewpoint sampling (host side of the GT-PVS generator).

Restates the reference's geometry on plain Python floats, operation for
operation, so camera bases come out bit-identical to the reference's and the
device GT-PVS (``gtpvs.py``) can be pinned bit-exactly:

* ``Vec3`` arithmetic, ``normalized`` = v * (1/sqrt(v.v)) (core.py:26-77);
* ``rotate_about`` (Rodrigues, core.py:79-85), ``Camera.from_forward`` /
  ``yawed`` (core.py:229-243), ``ViewCell.from_forward`` /
  ``displacement`` / ``camera_at`` (core.py:276-294);
* ``build_viewcell_frustum`` (core.py:361-373);
* ``sample_viewpoints`` — golden-angle spiral with van der Corput yaw, or
  seeded uniform draws (oracle.py:64-104).

Every function also accepts the reference's own objects (duck-typed:
anything with ``x, y, z`` is a vector), so reference callers pass their
``ViewCell`` / ``Camera`` unchanged.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

GOLDEN_ANGLE = math.pi * (3.0 - math.sqrt(5.0))


def _v(a):
    """(x, y, z) floats of a Vec3-like or a sequence."""
    if hasattr(a, "x"):
        return (float(a.x), float(a.y), float(a.z))
    x, y, z = (float(c) for c in a)
    return (x, y, z)


def add(a, b):
    return (a[0] + b[0], a[1] + b[1], a[2] + b[2])


def sub(a, b):
    return (a[0] - b[0], a[1] - b[1], a[2] - b[2])


def mul(a, s):
    return (a[0] * s, a[1] * s, a[2] * s)


def dot(a, b):
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]


def cross(a, b):
    return (a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0])


def norm(a):
    return math.sqrt(dot(a, a))


def normalized(a):
    n = norm(a)
    if n == 0.0:
        raise ValueError("cannot normalize a zero vector")
    return mul(a, 1.0 / n)


def rotate_about(v, axis, angle_deg):
    """core.py:79-85."""
    a = math.radians(angle_deg)
    k = normalized(axis)
    c, s = math.cos(a), math.sin(a)
    return add(add(mul(v, c), mul(cross(k, v), s)), mul(k, dot(k, v) * (1.0 - c)))


@dataclass
class Camera:
    """Pinhole camera (core.py:205-248): position, orthonormal (forward, up, right)."""

    position: tuple
    forward: tuple
    up: tuple
    right: tuple
    fov_deg: float
    near: float
    far: float

    @classmethod
    def of(cls, cam) -> "Camera":
        return cls(_v(cam.position), _v(cam.forward), _v(cam.up), _v(cam.right), float(cam.fov_deg),
                   float(cam.near), float(cam.far))

    @classmethod
    def from_forward(cls, position, forward, fov_deg, near, far, up_hint=(0.0, 1.0, 0.0)) -> "Camera":
        f = normalized(_v(forward))
        r = cross(f, _v(up_hint))
        if norm(r) < 1e-9:
            r = cross(f, (1.0, 0.0, 0.0))
        r = normalized(r)
        u = normalized(cross(r, f))
        return cls(_v(position), f, u, r, float(fov_deg), float(near), float(far))

    def yawed(self, angle_deg: float) -> "Camera":
        f = rotate_about(self.forward, self.up, -angle_deg)
        r = rotate_about(self.right, self.up, -angle_deg)
        return Camera(self.position, f, self.up, r, self.fov_deg, self.near, self.far)

    @property
    def half_extent(self) -> float:
        return math.tan(math.radians(self.fov_deg) / 2.0)

    def params(self):
        """(origin, basis rows right/up/forward, half_extent, near, far) as the raster takes them."""
        return self.position, (self.right, self.up, self.forward), self.half_extent, self.near, self.far


@dataclass
class ViewCell:
    """core.py:251-294."""

    center: tuple
    radius: float
    fov_deg: float
    beta_deg: float
    forward: tuple
    up: tuple
    right: tuple
    near: float
    far: float

    def __post_init__(self):
        if self.radius <= 0:
            raise ValueError("viewcell radius must be positive")
        if self.fov_deg + 2 * self.beta_deg >= 180.0:
            raise ValueError("enlarged fov (fov + 2*beta) must stay below 180 degrees")

    @classmethod
    def of(cls, cell) -> "ViewCell":
        if isinstance(cell, cls):
            return cell
        return cls(_v(cell.center), float(cell.radius), float(cell.fov_deg), float(cell.beta_deg),
                   _v(cell.forward), _v(cell.up), _v(cell.right), float(cell.near), float(cell.far))

    @classmethod
    def from_forward(cls, center, radius, fov_deg, beta_deg, forward, near, far,
                     up_hint=(0.0, 1.0, 0.0)) -> "ViewCell":
        cam = Camera.from_forward(center, forward, fov_deg, near, far, up_hint)
        return cls(_v(center), float(radius), float(fov_deg), float(beta_deg), cam.forward, cam.up, cam.right,
                   float(near), float(far))

    @property
    def displacement(self) -> float:
        return self.radius / math.tan(math.radians(self.fov_deg) / 2.0)

    @property
    def displaced_origin(self):
        return sub(self.center, mul(self.forward, self.displacement))

    def camera_at(self, position, yaw_deg: float = 0.0) -> Camera:
        cam = Camera(_v(position), self.forward, self.up, self.right, self.fov_deg, self.near, self.far)
        return cam.yawed(yaw_deg) if yaw_deg else cam


def build_viewcell_frustum(cell):
    """core.py:361-373 -> froxelize.Frustum."""
    from .froxelize import Frustum
    cell = ViewCell.of(cell)
    if cell.fov_deg + 2 * cell.beta_deg >= 180.0:
        raise ValueError("enlarged fov (fov + 2*beta) must stay below 180 degrees")
    disp = cell.displacement
    return Frustum.from_vectors(cell.displaced_origin, cell.forward, cell.up, cell.right,
                                cell.fov_deg + 2 * cell.beta_deg, disp, disp + cell.far)


def _vdc(i: int) -> float:
    x, f = 0.0, 0.5
    while i:
        x += f * (i & 1)
        i >>= 1
        f *= 0.5
    return x


def sample_viewpoints(cell, viewpoints: int = 128, mode: str = "uniform-grid", seed: int = 0) -> list:
    """oracle.py:64-104: ``viewpoints`` cameras over the cell's disc and yaw range."""
    cell = ViewCell.of(cell)
    m = int(viewpoints)
    if m < 1:
        raise ValueError("viewpoint count must be >= 1")
    if mode not in ("uniform-grid", "uniform-random"):
        raise ValueError(f"unknown sampling mode {mode!r}")
    if m == 1:
        return [cell.camera_at(cell.center, 0.0)]
    cams = []
    if mode == "uniform-grid":
        for i in range(m):
            rad = cell.radius * math.sqrt((i + 0.5) / m)
            ang = i * GOLDEN_ANGLE
            pos = add(add(cell.center, mul(cell.right, rad * math.cos(ang))), mul(cell.up, rad * math.sin(ang)))
            yaw = cell.beta_deg * (2.0 * _vdc(i + 1) - 1.0)
            cams.append(cell.camera_at(pos, yaw))
    else:
        rng = np.random.Generator(np.random.PCG64(seed))
        for _ in range(m):
            rad = cell.radius * math.sqrt(rng.random())
            ang = 2.0 * math.pi * rng.random()
            yaw = cell.beta_deg * (2.0 * rng.random() - 1.0)
            pos = add(add(cell.center, mul(cell.right, rad * math.cos(ang))), mul(cell.up, rad * math.sin(ang)))
            cams.append(cell.camera_at(pos, yaw))
    return cams
