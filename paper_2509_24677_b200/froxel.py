"""FPVS packed-occupancy grids: the byte format on both sides of the hot path.

Mirrors the reference's ``FroxelGrid`` (pkg/src/froxelpvs/froxel.py:64-196):

* bits are packed eight per byte along x, least significant bit first, with
  ``byte = (x >> 3) + (Nx/8) * (y + Ny*z)`` and ``bit = x & 7``
  (froxel.py:3-4, 96-104);
* ``Nx % 8 == 0`` is enforced (froxel.py:71-72);
* the FPVS file is a 24-byte header ``b"FPVS" <u32 version> <u32 Nx,Ny,Nz>
  <u8 role> <u8 supersample> <2 pad>`` followed by the packed bytes
  (froxel.py:178-196).

This class is host-side plumbing (numpy bytes).  The packed layout is also the
device layout: ``bits`` uploaded as-is is what the interleave kernel reads and
what the head kernel writes, so a grid crosses PCIe as Nx*Ny*Nz/8 bytes.
"""

from __future__ import annotations

import struct

import numpy as np

FPVS_MAGIC = b"FPVS"
FPVS_VERSION = 1
ROLE_TAGS = ("geometry", "gt_pvs", "predicted_pvs")


class FroxelGrid:
    """Binary occupancy over an (Nx, Ny, Nz) grid, packed x-fastest LSB-first."""

    def __init__(self, dims, role: str = "geometry", supersample: int = 1, bits=None):
        nx, ny, nz = (int(v) for v in dims)
        if min(nx, ny, nz) <= 0:
            raise ValueError("grid dims must be positive")
        if nx % 8:
            raise ValueError(f"N_x must be divisible by 8, got {nx}")
        if role not in ROLE_TAGS:
            raise ValueError(f"unknown role {role!r}")
        self.dims = (nx, ny, nz)
        self.role = role
        self.supersample = int(supersample)
        n = nx * ny * nz // 8
        if bits is None:
            self.bits = np.zeros(n, np.uint8)
        else:
            self.bits = np.ascontiguousarray(np.asarray(bits, dtype=np.uint8).reshape(-1))
            if self.bits.size != n:
                raise ValueError("bit buffer size does not match dims")

    @property
    def row_bytes(self) -> int:
        return self.dims[0] // 8

    def _byte_bit(self, x, y, z):
        nx, ny, nz = self.dims
        if not (0 <= x < nx and 0 <= y < ny and 0 <= z < nz):
            raise IndexError(f"froxel coordinate {(x, y, z)} out of range for dims {self.dims}")
        return (x >> 3) + self.row_bytes * (y + ny * z), x & 7

    def set(self, x: int, y: int, z: int):
        i, b = self._byte_bit(x, y, z)
        self.bits[i] |= np.uint8(1 << b)

    def get(self, x: int, y: int, z: int) -> int:
        i, b = self._byte_bit(x, y, z)
        return int(self.bits[i] >> b) & 1

    def to_dense(self) -> np.ndarray:
        """Boolean (Nx, Ny, Nz) view, C-order (z fastest)."""
        nx, ny, nz = self.dims
        planes = np.unpackbits(self.bits.reshape(nz, ny, nx // 8), axis=2, bitorder="little")
        return np.ascontiguousarray(planes.astype(bool).transpose(2, 1, 0))

    @classmethod
    def from_dense(cls, dense, role: str = "geometry", supersample: int = 1) -> "FroxelGrid":
        occ = np.asarray(dense).astype(bool)
        if occ.ndim != 3:
            raise ValueError("dense occupancy must be 3-dimensional")
        g = cls(occ.shape, role=role, supersample=supersample)
        g.bits = np.ascontiguousarray(
            np.packbits(occ.transpose(2, 1, 0), axis=2, bitorder="little").reshape(-1))
        return g

    def occupied_count(self) -> int:
        return int(np.unpackbits(self.bits).sum())

    def occupancy(self) -> float:
        nx, ny, nz = self.dims
        return self.occupied_count() / float(nx * ny * nz)

    def copy(self) -> "FroxelGrid":
        return FroxelGrid(self.dims, self.role, self.supersample, self.bits.copy())

    def subset_of(self, other: "FroxelGrid") -> bool:
        if self.dims != other.dims:
            raise ValueError(f"grid dims mismatch: {self.dims} vs {other.dims}")
        return not np.any(self.bits & ~other.bits)

    def __eq__(self, other):
        if not isinstance(other, FroxelGrid):
            return NotImplemented
        return (self.dims == other.dims and self.role == other.role
                and np.array_equal(self.bits, other.bits))

    def save(self, path):
        head = FPVS_MAGIC + struct.pack("<IIIIBBxx", FPVS_VERSION, *self.dims,
                                        ROLE_TAGS.index(self.role), self.supersample & 0xFF)
        with open(path, "wb") as fh:
            fh.write(head + self.bits.tobytes())

    @classmethod
    def load(cls, path) -> "FroxelGrid":
        with open(path, "rb") as fh:
            raw = fh.read()
        if raw[:4] != FPVS_MAGIC:
            raise ValueError(f"{path}: not an FPVS grid file")
        version, nx, ny, nz, role, ss = struct.unpack_from("<IIIIBB", raw, 4)
        if version != FPVS_VERSION:
            raise ValueError(f"{path}: unsupported FPVS version {version}")
        return cls((nx, ny, nz), ROLE_TAGS[role], ss, np.frombuffer(raw, np.uint8, offset=24).copy())
