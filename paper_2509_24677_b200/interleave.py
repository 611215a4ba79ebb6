"""Drop-in ``interleave`` / ``deinterleave`` backed by the CUDA kernels.

Mirrors pkg/src/froxelpvs/interleave.py:18-85:

* ``ChannelTensor(values, d)`` — 4-D channels-last, channels == d^3
  (interleave.py:18-42), ValueError otherwise;
* ``interleave(grid, d)`` — FroxelGrid -> float64 values, ndarray keeps its
  dtype, 3-D only, non-divisible dims -> ValueError (interleave.py:45-65);
* ``deinterleave(t, d=None, threshold=None, role=...)`` — exact inverse; with
  a threshold applies ``>= tau`` and returns a packed FroxelGrid
  (interleave.py:68-85).

Values move exactly: float64 (and integer) arrays are permuted as 8-byte
elements on the device, float32 and u8 as themselves, and a threshold is
compared in the cells' own precision (float64 cells in float64).

The arithmetic runs on the GPU (``fpvs_interleave`` / ``fpvs_deinterleave``).
numpy/FroxelGrid inputs are copied to the device and the result copied back,
so reference-style callers get numpy out; CUDA tensors stay on the device and
may carry a leading batch dimension (B, Nx, Ny, Nz).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .froxel import FroxelGrid


@dataclass
class ChannelTensor:
    """Interleaved grid: spatial dims (N_x/d, N_y/d, N_z/d), d^3 channels last."""

    values: object
    d: int

    def __post_init__(self):
        shape = tuple(self.values.shape)
        if len(shape) != 4:
            raise ValueError("channel tensor must be 4-dimensional (x, y, z, channels)")
        if shape[3] != self.d ** 3:
            raise ValueError(f"channel count {shape[3]} does not match d^3 = {self.d ** 3}")

    @property
    def spatial_dims(self) -> tuple:
        return tuple(self.values.shape[:3])

    @property
    def channels(self) -> int:
        return int(self.values.shape[3])

    @property
    def grid_dims(self) -> tuple:
        return tuple(int(s) * self.d for s in self.values.shape[:3])


def _torch():
    import torch
    return torch


def interleave_device(grid, d: int, out_dtype=None, packed_dims=None, want_active: bool = False):
    """Batched device interleave.

    ``grid``: CUDA tensor (B, Nx, Ny, Nz) float32/uint8/bool, or packed uint8
    bits of B grids with ``packed_dims=(B, Nx, Ny, Nz)``.  Returns the
    (B, X, Y, Z, d^3) tensor (and the u8 cell-active mask when asked).
    """
    torch = _torch()
    if packed_dims is not None:
        B, nx, ny, nz = packed_dims
        fmt, src = _lib.IN_PACKED, grid.contiguous()
    else:
        if grid.dim() != 4:
            raise ValueError("expected a (B, Nx, Ny, Nz) tensor")
        B, nx, ny, nz = grid.shape
        if grid.dtype in (torch.bool, torch.uint8):
            fmt, src = _lib.IN_U8, grid.to(torch.uint8).contiguous()
        elif grid.dtype == torch.float64:
            fmt, src = _lib.IN_F64, grid.contiguous()
        else:
            fmt, src = _lib.IN_F32, grid.to(torch.float32).contiguous()
    if d < 1 or nx % d or ny % d or nz % d:
        raise ValueError(f"interleave factor {d} must divide grid dims {(nx, ny, nz)}")
    if fmt == _lib.IN_F64:
        out_dtype = torch.float64  # exact permutation of the float64 values
    out_dtype = out_dtype or torch.float32
    od = {torch.bfloat16: _lib.BF16, torch.float64: _lib.F64}.get(out_dtype, _lib.F32)
    out = torch.empty((B, nx // d, ny // d, nz // d, d ** 3), dtype=out_dtype, device=src.device)
    act = torch.empty((B, nx // d, ny // d, nz // d), dtype=torch.uint8, device=src.device) if want_active else None
    _lib.call("fpvs_interleave", _lib.ptr(src), fmt, B, nx, ny, nz, d, _lib.ptr(out), od, _lib.ptr(act),
              _lib.stream_ptr())
    return (out, act) if want_active else out


def interleave(grid, d: int) -> ChannelTensor:
    """Repack d x d x d froxel blocks into d^3-channel cells (interleave.py:54-65)."""
    torch = _torch()
    _lib.require_cuda()
    if isinstance(grid, FroxelGrid):
        nx, ny, nz = grid.dims
        if d < 1 or nx % d or ny % d or nz % d:
            raise ValueError(f"interleave factor {d} must divide grid dims {(nx, ny, nz)}")
        bits = torch.from_numpy(grid.bits).cuda()
        out = interleave_device(bits, d, torch.float32, packed_dims=(1, nx, ny, nz))
        return ChannelTensor(out[0].cpu().numpy().astype(np.float64), d)
    if isinstance(grid, torch.Tensor):
        if grid.dim() != 3:
            raise ValueError("expected a FroxelGrid or a dense 3D array")
        dt = grid.dtype
        src = grid if dt in (torch.bool, torch.uint8, torch.float32, torch.float64) else grid.to(torch.float64)
        out = interleave_device(src[None].cuda(), d, torch.float32)[0]
        return ChannelTensor(out.to(dt if dt.is_floating_point else torch.float32), d)
    arr = np.asarray(grid)
    if arr.ndim != 3:
        raise ValueError("expected a FroxelGrid or a dense 3D array")
    nx, ny, nz = arr.shape
    if d < 1 or nx % d or ny % d or nz % d:
        raise ValueError(f"interleave factor {d} must divide grid dims {(nx, ny, nz)}")
    # the reference keeps the input dtype (interleave.py:45-51), so the values
    # must move unchanged: u8/bool and float32 travel as themselves, float64
    # (and every other dtype, through float64: exact for integers < 2^53) as
    # float64 — the device permutes the 8-byte elements exactly
    if arr.dtype in (np.bool_, np.uint8):
        src = torch.from_numpy(np.ascontiguousarray(arr.astype(np.uint8)))[None].cuda()
    elif arr.dtype == np.float32:
        src = torch.from_numpy(np.ascontiguousarray(arr))[None].cuda()
    else:
        src = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64))[None].cuda()
    out = interleave_device(src, d, torch.float32)[0].cpu().numpy()
    return ChannelTensor(out.astype(arr.dtype, copy=False), d)


def deinterleave_device(cells, d: int, threshold: float | None = None):
    """Batched device deinterleave of (B, X, Y, Z, d^3) -> dense f32 or packed bits."""
    torch = _torch()
    if cells.dim() != 5 or cells.shape[4] != d ** 3:
        raise ValueError(f"channel count {cells.shape[-1]} does not match d^3 = {d ** 3}")
    B, X, Y, Z, _ = cells.shape
    src = cells.contiguous()
    if src.dtype not in (torch.float32, torch.bfloat16, torch.float64):
        src = src.to(torch.float64)
    dt = {torch.bfloat16: _lib.BF16, torch.float64: _lib.F64}.get(src.dtype, _lib.F32)
    if threshold is None:
        odt = torch.float64 if src.dtype == torch.float64 else torch.float32
        out = torch.empty((B, X * d, Y * d, Z * d), dtype=odt, device=src.device)
        tau = float("nan")
    else:
        if (X * d) % 8:
            raise ValueError(f"N_x must be divisible by 8, got {X * d}")
        out = torch.empty(B * X * d * Y * d * Z * d // 8, dtype=torch.uint8, device=src.device)
        tau = float(threshold)
    _lib.call("fpvs_deinterleave", _lib.ptr(src), dt, B, X, Y, Z, d, tau, _lib.ptr(out), _lib.stream_ptr())
    return out


def deinterleave(tensor: ChannelTensor, d: int | None = None, threshold: float | None = None,
                 role: str = "predicted_pvs"):
    """Invert :func:`interleave` (interleave.py:68-85)."""
    torch = _torch()
    _lib.require_cuda()
    if d is None:
        d = tensor.d
    if d != tensor.d or tensor.channels != d ** 3:
        raise ValueError(f"channel count {tensor.channels} does not match d^3 = {d ** 3}")
    vals = tensor.values
    on_host = not isinstance(vals, torch.Tensor)
    if on_host:
        arr = np.asarray(vals)
        # float32 cells compare in float32 and float64 in float64, as the
        # reference's numpy `values >= threshold` does (NEP 50)
        keep = arr.dtype if arr.dtype in (np.float32, np.float64) else np.float64
        src = torch.from_numpy(np.ascontiguousarray(arr, dtype=keep)).cuda()
    else:
        src = vals.cuda()
    if threshold is None:
        out = deinterleave_device(src[None], d)[0]
        if on_host:
            return out.cpu().numpy().astype(np.asarray(vals).dtype, copy=False)
        return out
    bits = deinterleave_device(src[None], d, threshold)
    return FroxelGrid(tensor.grid_dims, role=role, bits=bits.cpu().numpy())
