"""torch ``nn.Module`` / ``autograd.Function`` face of the path (BASELINE north star).

The reference's layer API is numpy with hand-written backward passes
(Conv3d.forward / Conv3d.backward, neural.py:201-249; PvsNet, neural.py:
260-297; combined_loss, neural.py:395-399).  These wrappers expose the same
operations to torch autograd so a standard torch training loop works
unchanged (``loss.backward(); torch.optim.AdamW(...).step()``), every op
running in libfpvs:

* ``SparseConv3dFunction`` — forward ``fpvs_spconv_simt`` (fp32, fused bias
  + activation); backward ``fpvs_spconv_wgrad_simt`` (dW, db; deterministic)
  and ``fpvs_spconv_dgrad_simt`` (dx over the mirrored map).  The relu' of
  the layer's own output (z > 0 <=> y > 0, neural.py:227-228) masks the
  incoming gradient first.
* ``PvsLossFunction`` — ``combined_loss`` (dice + repulsive visibility,
  batch mean) from ``fpvs_loss_counts`` / ``fpvs_loss_grad`` on the head
  logits; its backward is the fused dL/dlogit.
* ``SparseConv3d`` / ``PvsNetModule`` — Parameters in the reference layout
  ((k^3 Cin, Cout) rows ((a k + b) k + c) Cin + ci, neural.py:163-166),
  initialised exactly like ``neural.PvsNet``; ``PvsNetModule.forward``
  builds the sparse level from packed grids (fused level build) and returns
  the head logits per active cell.

``precision="bf16"`` runs layers with Cout % 32 == 0 through
``SparseConv3dTCFunction`` (tcgen05 forward, wgrad and dgrad; bf16 rows,
fp32 Parameters and gradients); the rest stay on the fp32 kernels.

Rows are the active cells of a ``sparse.Level`` (C-order, capacity ``cap``,
count ``n`` on the device); rows past ``n`` are zero in every output and
gradient.  The fused, graph-friendly bf16 training step is
``train.TrainStep``.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from . import sparse as sp
from .neural import ModelConfig, PvsNet, TrainConfig


def _torch():
    import torch
    return torch


def _nn():
    import torch.nn as nn
    return nn


def _table(level, K):
    return (level.nbr, 27) if K == 27 else (None, 1)


def _make_conv_fn():
    torch = _torch()

    class SparseConv3dFunction(torch.autograd.Function):
        """y = act(conv(x) + b) on the active rows of ``level`` (neural.py:201-219)."""

        @staticmethod
        def forward(ctx, x, w, b, level, K: int, act: str):
            cap, cin = x.shape
            cout = w.shape[1]
            ctx.in_dtype = x.dtype
            x = x.contiguous().float()
            y = torch.zeros((cap, cout), dtype=torch.float32, device=x.device)
            table, K = _table(level, K)
            _lib.call("fpvs_spconv_simt", _lib.ptr(x), cin, _lib.F32, _lib.ptr(table), K, _lib.ptr(level.n), cap,
                      _lib.ptr(w.detach().contiguous()), _lib.ptr(b.detach().contiguous()), cin, cout,
                      _lib.ACT[act], _lib.ptr(y), cout, 0, _lib.F32, _lib.stream_ptr())
            ctx.save_for_backward(x, w, y)
            ctx.level, ctx.K, ctx.act = level, K, act
            return y

        @staticmethod
        def backward(ctx, dy):
            x, w, y = ctx.saved_tensors
            level, K, act = ctx.level, ctx.K, ctx.act
            cap, cin = x.shape
            cout = w.shape[1]
            dz = dy.contiguous().float()
            if act == "relu":
                dz = torch.where(y > 0, dz, torch.zeros_like(dz))  # relu' with z > 0 (neural.py:227-228)
            elif act == "sigmoid":
                dz = dz * y * (1.0 - y)  # sigmoid' = y(1 - y) (neural.py:229-230)
            table, K = _table(level, K)
            s = _lib.stream_ptr()
            dw = torch.empty_like(w, dtype=torch.float32)
            db = torch.empty(cout, dtype=torch.float32, device=x.device)
            ws = torch.empty(_lib.size("fpvs_wgrad_workspace_size", K, cin, cout, cap), dtype=torch.uint8,
                             device=x.device)
            _lib.call("fpvs_spconv_wgrad_simt", _lib.ptr(x), cin, _lib.F32, _lib.ptr(dz), cout, _lib.ptr(table), K,
                      _lib.ptr(level.n), cap, cin, cout, _lib.ptr(dw), _lib.ptr(db), _lib.ptr(ws), ws.numel(), s)
            dx = None
            if ctx.needs_input_grad[0]:
                dx = torch.zeros((cap, cin), dtype=torch.float32, device=x.device)
                _lib.call("fpvs_spconv_dgrad_simt", _lib.ptr(dz), cout, _lib.ptr(table), K, _lib.ptr(level.n), cap,
                          _lib.ptr(w.detach().contiguous()), cin, cout, None, 0, 0, _lib.ptr(dx), cin, s)
                dx = dx.to(ctx.in_dtype)
            return dx, dw, db, None, None, None

    return SparseConv3dFunction


def _make_conv_tc_fn():
    torch = _torch()
    from .neural import pack_tc

    class SparseConv3dTCFunction(torch.autograd.Function):
        """bf16 tensor-core version: forward fpvs_spconv_tc (weights packed from the
        fp32 Parameter each call), backward fpvs_spconv_wgrad_tc + fpvs_spconv_tc_dgrad."""

        @staticmethod
        def forward(ctx, x, w, b, level, K: int, act: str):
            cap, cin = x.shape
            cout = w.shape[1]
            x = x.contiguous().to(torch.bfloat16)
            y = torch.zeros((cap, cout), dtype=torch.bfloat16, device=x.device)
            table, K = _table(level, K)
            masks = level.nbr_masks if table is not None else None
            if table is not None and masks is None:
                masks = sp.tile_masks(table, K, level.n, cap)
            packed = pack_tc(w.detach(), K, cin, cout, 0)
            _lib.call("fpvs_spconv_tc", _lib.ptr(x), cin, cap, _lib.ptr(table), K, _lib.ptr(masks),
                      _lib.ptr(level.n), cap, _lib.ptr(packed), 0, _lib.ptr(b.detach().contiguous()), cin, cout,
                      _lib.ACT[act], _lib.ptr(y), cout, 0, _lib.stream_ptr())
            ctx.save_for_backward(x, w, y)
            ctx.level, ctx.K, ctx.act, ctx.masks = level, K, act, masks
            return y

        @staticmethod
        def backward(ctx, dy):
            x, w, y = ctx.saved_tensors
            level, K, act, masks = ctx.level, ctx.K, ctx.act, ctx.masks
            cap, cin = x.shape
            cout = w.shape[1]
            dz = dy
            if act == "relu":
                dz = torch.where(y > 0, dz, torch.zeros_like(dz))  # relu' with z > 0 (neural.py:227-228)
            elif act == "sigmoid":
                yf = y.float()
                dz = dz.float() * yf * (1.0 - yf)
            dz = dz.to(torch.bfloat16).contiguous()
            table, K = _table(level, K)
            s = _lib.stream_ptr()
            dw = torch.empty(w.shape, dtype=torch.float32, device=x.device)
            db = torch.empty(cout, dtype=torch.float32, device=x.device)
            ws = torch.empty(_lib.size("fpvs_wgrad_tc_workspace_size", K, cin, cout, cap), dtype=torch.uint8,
                             device=x.device)
            _lib.call("fpvs_spconv_wgrad_tc", _lib.ptr(x), cin, _lib.ptr(dz), cout, _lib.ptr(table), K,
                      _lib.ptr(level.n), cap, cin, cout, _lib.ptr(dw), _lib.ptr(db), _lib.ptr(ws), ws.numel(), s)
            dx = None
            if ctx.needs_input_grad[0]:
                if cin % 32:
                    raise ValueError(f"tensor-core dgrad needs Cin % 32 == 0, got {cin}")
                nbytes = _lib.size("fpvs_pack_weights_tc_size", K, cout, cin, 0)
                pd = torch.empty(nbytes, dtype=torch.uint8, device=x.device)
                _lib.call("fpvs_pack_weights_tc_dgrad", _lib.ptr(w.detach().contiguous()), K, cin, cout, 0,
                          _lib.ptr(pd), s)
                dx = torch.zeros((cap, cin), dtype=torch.bfloat16, device=x.device)
                _lib.call("fpvs_spconv_tc_dgrad", _lib.ptr(dz), cout, cap, _lib.ptr(table), K, _lib.ptr(masks),
                          _lib.ptr(level.n), cap, _lib.ptr(pd), 0, cin, cout, None, 0, _lib.ptr(dx), cin, s)
            return dx, dw, db, None, None, None

    return SparseConv3dTCFunction


def _make_loss_fn():
    torch = _torch()

    class PvsLossFunction(torch.autograd.Function):
        """combined_loss (neural.py:395-399) of sigmoid(logits) against packed labels, batch mean."""

        @staticmethod
        def forward(ctx, logits, level, gt_bits, grid_dims, d: int, alpha: float, lam: float):
            cap, c = logits.shape
            nx, ny, nz = grid_dims
            probs = torch.sigmoid(logits.detach().float()).contiguous()
            s = _lib.stream_ptr()
            sums = torch.empty((_lib.size("fpvs_loss_sums_size", level.B, cap) + 7) // 8, dtype=torch.float64,
                               device=logits.device)
            dlog = torch.zeros((cap, c), dtype=torch.float32, device=logits.device)
            loss = torch.zeros(1, dtype=torch.float64, device=logits.device)
            _lib.call("fpvs_loss_counts", _lib.ptr(probs), c, _lib.ptr(level.coords), _lib.ptr(level.n), cap,
                      _lib.ptr(gt_bits), d, level.B, nx, ny, nz, _lib.ptr(sums), s)
            _lib.call("fpvs_loss_grad", _lib.ptr(probs), c, _lib.ptr(level.coords), _lib.ptr(level.n), cap,
                      _lib.ptr(gt_bits), d, level.B, nx, ny, nz, _lib.ptr(sums), float(alpha), float(lam),
                      _lib.ptr(dlog), _lib.ptr(loss), s)
            ctx.save_for_backward(dlog)
            ctx.logit_dtype = logits.dtype
            return loss[0]

        @staticmethod
        def backward(ctx, g):
            (dlog,) = ctx.saved_tensors
            return (dlog * g.float()).to(ctx.logit_dtype), None, None, None, None, None, None

    return PvsLossFunction


_FNS = {}


def sparse_conv3d(x, w, b, level, K: int, act: str, precision: str = "fp32"):
    """Differentiable submanifold conv on the active rows of ``level`` (fp32 SIMT
    or bf16 tensor cores)."""
    # tensor cores need Cout % 32 == 0 (store epilogue); e.g. the d^3 = 8 head stays fp32
    tc = precision == "bf16" and w.shape[1] % 32 == 0
    key = "conv_tc" if tc else "conv"
    if key not in _FNS:
        _FNS[key] = _make_conv_tc_fn() if tc else _make_conv_fn()
    return _FNS[key].apply(x, w, b, level, K, act)


def pvs_loss(logits, level, gt_bits, grid_dims, d: int, alpha: float = 0.1, lam: float = 0.99):
    """Differentiable combined loss (batch mean, float64 scalar)."""
    if "loss" not in _FNS:
        _FNS["loss"] = _make_loss_fn()
    return _FNS["loss"].apply(logits, level, gt_bits, tuple(grid_dims), d, alpha, lam)


def SparseConv3d(spec, rng: np.random.Generator | None = None, init: str = "he", device: str = "cuda"):
    """nn.Module with ``weight`` (k^3 Cin, Cout) and ``bias`` Parameters (reference layout)."""
    nn = _nn()
    from .neural import Conv3d

    class _SparseConv3d(nn.Module):
        def __init__(self):
            super().__init__()
            ref = Conv3d(spec, rng, init, device)
            self.spec = spec
            self.weight = nn.Parameter(ref.w.clone())
            self.bias = nn.Parameter(ref.b.clone())

        def forward(self, x, level):
            return sparse_conv3d(x, self.weight, self.bias, level, self.spec.kernel ** 3, self.spec.activation)

    return _SparseConv3d()


class PvsNetModule:
    """Factory for the torch module of a linear ``ModelConfig`` network (neural.py:260-297)."""

    def __new__(cls, cfg: ModelConfig, rng: np.random.Generator | None = None, device: str = "cuda",
                precision: str = "fp32"):
        nn = _nn()
        torch = _torch()
        _lib.require_cuda()
        ref = PvsNet(cfg, rng, device=device, precision="fp32")

        class _PvsNetModule(nn.Module):
            def __init__(self):
                super().__init__()
                self.cfg = cfg
                self.precision = precision
                self.layers = nn.ModuleList()
                for L in ref.layers:
                    m = SparseConv3d(L.spec, None, device=device)
                    with torch.no_grad():
                        m.weight.copy_(L.w)
                        m.bias.copy_(L.b)
                    self.layers.append(m)
                self._levels = {}

            def level(self, bits, B: int, grid_dims):
                """Sparse level + level-0 features of B packed grids (fused build, reused per shape)."""
                key = (B, tuple(grid_dims))
                d = self.cfg.d
                if key not in self._levels:
                    nx, ny, nz = grid_dims
                    lv = sp.new_level(B, (nx // d, ny // d, nz // d), device=bits.device)
                    maps = sp.LevelMaps([lv], [], [], tuple(grid_dims), d)
                    fdt = torch.float32 if self.precision == "fp32" else torch.bfloat16
                    feat = torch.zeros((lv.cap, d ** 3), dtype=fdt, device=bits.device)
                    self._levels[key] = (lv, maps, feat)
                lv, maps, feat = self._levels[key]
                maps.run(bits, feat)
                return lv, feat

            def forward(self, bits, B: int, grid_dims):
                """Head logits [cap, d^3] per active cell (rows past n are zero) and the level."""
                lv, x = self.level(bits, B, grid_dims)
                for i, m in enumerate(self.layers):
                    act = "none" if i == len(self.layers) - 1 else m.spec.activation
                    x = sparse_conv3d(x, m.weight, m.bias, lv, m.spec.kernel ** 3, act, self.precision)
                return x, lv

            def loss(self, bits, gt_bits, B: int, grid_dims, tcfg: TrainConfig | None = None):
                """combined_loss of one batch (neural.py:472-477), differentiable."""
                tcfg = tcfg or TrainConfig()
                logits, lv = self.forward(bits, B, grid_dims)
                return pvs_loss(logits, lv, gt_bits, grid_dims, self.cfg.d, tcfg.alpha, tcfg.lam)

        return _PvsNetModule()
