"""Drop-in NeuralPVS estimator API (pkg/src/froxelpvs/neural.py) on B200 kernels.

Same names, argument order and error behaviour as the reference:
``ConvSpec``, ``ModelConfig``, ``TrainConfig``, ``ConfusionCounts``,
``TrainingDiverged``, ``Conv3d``, ``PvsNet`` (forward / save / load, FPVW),
``dice_loss``, ``rvl_loss``, ``combined_loss``, ``predict_pvs``; ``train`` lives
in ``paper_2509_24677_b200.train`` and is re-exported here.

Semantics: the convolution is SUBMANIFOLD — outputs exist on the active cells
(any nonzero channel) and inactive cells read as zero / predict p = 0.  This is
the masked form of the reference's dense Conv3d (neural.py:201-219) that
SURVEY.md §7.3 item 5 fixes as the parity target; the unmasked dense
reference is not.

Numerics: ``precision="fp32"`` runs the SIMT FFMA kernels (logits within 1e-4
of the float64 oracle); ``precision="bf16"`` runs the tcgen05 kernels (bf16
activations and weights, fp32 accumulation in TMEM).
"""

from __future__ import annotations

import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _lib
from . import sparse as sp
from .froxel import FroxelGrid

FPVW_MAGIC = b"FPVW"
FPVW_VERSION = 1
ACTIVATIONS = ("relu", "sigmoid", "none")
INITS = ("he", "identity", "kaiming_uniform")


def _torch():
    import torch
    return torch


class TrainingDiverged(RuntimeError):
    """Raised when a non-finite loss shows up; carries the batch index (neural.py:30-35)."""

    def __init__(self, batch_index: int, value: float):
        super().__init__(f"non-finite loss {value!r} at batch {batch_index}")
        self.batch_index = batch_index


# ---------------------------------------------------------------------------
# configuration (neural.py:42-127)
# ---------------------------------------------------------------------------

@dataclass
class ConvSpec:
    kernel: int
    in_channels: int
    out_channels: int
    activation: str = "relu"

    def __post_init__(self):
        if self.kernel < 1 or self.kernel % 2 == 0:
            raise ValueError("kernel size must be odd so spatial dims are preserved")
        if self.in_channels < 1 or self.out_channels < 1:
            raise ValueError("channel counts must be positive")
        if self.activation not in ACTIVATIONS:
            raise ValueError(f"unknown activation {self.activation!r}")


@dataclass
class ModelConfig:
    d: int
    layers: list
    init: str = "he"

    def __post_init__(self):
        if self.d < 1:
            raise ValueError("interleave factor must be >= 1")
        if not self.layers:
            raise ValueError("model needs at least one layer")
        if self.init not in INITS:
            raise ValueError(f"unknown init {self.init!r}")
        want = self.d ** 3
        if self.layers[0].in_channels != want:
            raise ValueError(f"first layer must take d^3 = {want} channels")
        for prev, cur in zip(self.layers, self.layers[1:]):
            if cur.in_channels != prev.out_channels:
                raise ValueError("layer channel chain is inconsistent")
        last = self.layers[-1]
        if last.out_channels != want or last.activation != "sigmoid":
            raise ValueError(f"final layer must emit d^3 = {want} channels with sigmoid")
        if self.init == "identity":
            for spec in self.layers:
                if spec.out_channels < want and spec is not self.layers[-1]:
                    raise ValueError("identity init needs >= d^3 channels per hidden layer")
        # any odd kernel (ConvSpec) and any head kernel run on the device: k = 3
        # on the tensor-core / halo kernels, other k on the SIMT gather-GEMM over
        # a k^3-tap map (fpvs_kmap_subm_k); a 1x1x1 head is fused with the
        # threshold and bit-pack, a wider head runs as a conv + fpvs_head_rows

    @classmethod
    def default(cls, d: int = 4, hidden: int = 32, init: str = "he") -> "ModelConfig":
        """The reference's default estimator (neural.py:94-99): two 3^3 ReLU
        convs and a 3^3 sigmoid head."""
        c = d ** 3
        return cls(d, [ConvSpec(3, c, hidden, "relu"), ConvSpec(3, hidden, hidden, "relu"),
                       ConvSpec(3, hidden, c, "sigmoid")], init)

    @classmethod
    def config1(cls, init: str = "kaiming_uniform") -> "ModelConfig":
        """BASELINE config 1: d=2; 4 x subm 3^3 at 32 ch + ReLU; 1^3 conv to 8 ch; sigmoid."""
        return cls(2, [ConvSpec(3, 8, 32, "relu")] + [ConvSpec(3, 32, 32, "relu") for _ in range(3)]
                   + [ConvSpec(1, 32, 8, "sigmoid")], init)


@dataclass
class TrainConfig:
    alpha: float = 0.1
    lam: float = 0.99
    tau: float = 0.5
    lr: float = 1e-3
    decay: float = 1e-10
    batch_size: int = 3
    epochs: int = 50
    seed: int = 0
    optimizer: str = "sgd"        # "sgd" (reference, neural.py:481) | "adamw" (BASELINE config 5)
    weight_decay: float = 0.01

    def __post_init__(self):
        for name in ("alpha", "lam", "tau"):
            v = getattr(self, name)
            if not 0.0 <= v <= 1.0:
                raise ValueError(f"{name} must lie in [0, 1], got {v}")
        if self.lr <= 0:
            raise ValueError("learning rate must be positive")
        if not 0.0 <= self.decay < 1.0:
            raise ValueError("decay must lie in [0, 1)")
        if self.batch_size < 1 or self.epochs < 0:
            raise ValueError("batch size must be >= 1 and epochs >= 0")
        if self.seed < 0:
            raise ValueError("seed must be nonnegative")
        if self.optimizer not in ("sgd", "adamw"):
            raise ValueError(f"unknown optimizer {self.optimizer!r}")


@dataclass
class ConfusionCounts:
    tp: float
    fp: float
    fn: float
    gtp: float

    @staticmethod
    def from_soft(pred, gt) -> "ConfusionCounts":
        """TP = sum p*g, FP = sum p*(1-g), FN = sum (1-p)*g, GTP = sum g (neural.py:139-144)."""
        p = _as_cuda64(pred)
        g = _as_cuda64(gt)
        tp = float((p * g).sum())
        ps = float(p.sum())
        gs = float(g.sum())
        return ConfusionCounts(tp, ps - tp, gs - tp, gs)


def _as_cuda64(a):
    torch = _torch()
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=torch.float64)
    return torch.as_tensor(np.asarray(a, dtype=np.float64), device="cuda")


# ---------------------------------------------------------------------------
# layers
# ---------------------------------------------------------------------------

class Conv3d:
    """Submanifold 3-D conv (k = 1 or 3) + bias + activation with device weights.

    ``w`` is the reference's (k^3 * Cin, Cout) matrix, row ((a*k + b)*k + c)*Cin
    + ci (neural.py:163-166), held as float32 on the GPU; ``packed()`` is the
    bf16 128B-swizzled image the tcgen05 kernel streams (built once).
    """

    def __init__(self, spec: ConvSpec, rng: np.random.Generator | None = None, init: str = "he",
                 device: str = "cuda"):
        torch = _torch()
        self.spec = spec
        k3c = spec.kernel ** 3 * spec.in_channels
        gain = 2.0 if spec.activation == "relu" else 1.0
        if rng is None:
            w = np.zeros((k3c, spec.out_channels))
        elif init == "kaiming_uniform":
            bound = np.sqrt(3.0 * gain / k3c)
            w = rng.uniform(-bound, bound, size=(k3c, spec.out_channels))
        else:  # reference He-normal draw (neural.py:174-175); identity re-seeds below
            w = rng.normal(0.0, np.sqrt(gain / k3c), size=(k3c, spec.out_channels))
        self.w = torch.tensor(w, dtype=torch.float32, device=device)
        self.b = torch.zeros(spec.out_channels, dtype=torch.float32, device=device)
        self._packed = None

    @property
    def taps(self) -> int:
        return self.spec.kernel ** 3

    def seed_identity(self, rng: np.random.Generator, gain: float, noise: float = 0.02):
        """Centre-tap identity plus small noise, drawn as neural.py:178-185."""
        torch = _torch()
        k3, cin, cout = self.taps, self.spec.in_channels, self.spec.out_channels
        w = rng.normal(0.0, noise / np.sqrt(k3 * cin), size=(k3, cin, cout))
        for j in range(min(cin, cout)):
            w[k3 // 2, j, j] += gain
        self.w = torch.tensor(w.reshape(k3 * cin, cout), dtype=torch.float32, device=self.w.device)
        self._packed = None

    def set_weights(self, w, b):
        torch = _torch()
        self.w = torch.as_tensor(np.asarray(w, dtype=np.float32) if not isinstance(w, torch.Tensor) else w,
                                 dtype=torch.float32).to(self.w.device).contiguous()
        self.b = torch.as_tensor(np.asarray(b, dtype=np.float32) if not isinstance(b, torch.Tensor) else b,
                                 dtype=torch.float32).to(self.w.device).contiguous()
        self._packed = None

    def invalidate(self):
        self._packed = None

    def packed(self, bn: int = 0, stream=None):
        return packed_cache(self, bn, stream)

    # -- reference-shaped dense API (neural.py:201-249) ----------------------
    def forward(self, x, keep_cache: bool = False, level: sp.Level | None = None):
        """(B, D, H, W, Cin) -> activation output (B, D, H, W, Cout); with
        ``keep_cache`` also the backward cache (neural.py:201-219).

        Submanifold: outputs exist on the active cells — those with any nonzero
        input channel, or the cells of ``level`` when a network passes its
        level-0 set along — and read 0 elsewhere.  fp32 on the device (SIMT
        FFMA); numpy in -> float64 numpy out, CUDA tensors stay on the device.
        """
        torch = _torch()
        host = not isinstance(x, torch.Tensor)
        xt = _dense_in(x, self.spec.in_channels)
        lv = level if level is not None else dense_level(xt)
        x_rows = dense_to_rows(xt, lv)
        y_rows = self.forward_rows_f32(x_rows, lv)
        y = rows_to_dense(y_rows, lv, self.spec.out_channels)
        out = y.cpu().numpy().astype(np.float64) if host else y
        if not keep_cache:
            return out
        return out, Conv3dCache(lv, x_rows, y_rows, tuple(xt.shape), host)

    def forward_rows_f32(self, x_rows, lv: sp.Level, stream=None):
        """fp32 rows in -> fp32 activation rows out on level ``lv``."""
        torch = _torch()
        build_layer_tables(lv, [self.spec.kernel], stream)
        table, K, _ = layer_table(lv, self.spec.kernel)
        y_rows = torch.zeros((lv.cap, self.spec.out_channels), dtype=torch.float32, device=x_rows.device)
        run_conv(self, x_rows, x_rows.shape[1], table, K, lv.n, lv.cap, y_rows, y_rows.shape[1], 0, "fp32",
                 stream=stream)
        return y_rows

    def backward(self, dy, cache):
        """Gradients (dx, dw, db) of the scalar loss (neural.py:221-249) on the
        cached active set: relu' = z > 0, sigmoid' = y (1 - y); dw in the
        reference's (k^3 Cin, Cout) row order."""
        if cache is None:
            raise ValueError("backward requires the forward cache")
        torch = _torch()
        host = not isinstance(dy, torch.Tensor)
        dyt = _dense_in(dy, self.spec.out_channels)
        if tuple(dyt.shape[:4]) != tuple(cache.shape[:4]):
            raise ValueError(f"gradient shape {tuple(dyt.shape)} does not match the cached output")
        dx_rows, dw, db = self.backward_rows(dense_to_rows(dyt, cache.level), cache)
        dx = rows_to_dense(dx_rows, cache.level, self.spec.in_channels)
        if host:
            return (dx.cpu().numpy().astype(np.float64), dw.cpu().numpy().astype(np.float64),
                    db.cpu().numpy().astype(np.float64))
        return dx, dw, db

    def backward_rows(self, dy_rows, cache, need_dx: bool = True, stream=None):
        """Rows form of :meth:`backward`: fpvs_act_backward, fpvs_spconv_wgrad_simt
        (deterministic) and fpvs_spconv_dgrad_simt (mirrored offsets)."""
        torch = _torch()
        lv, spec = cache.level, self.spec
        s = _lib.stream_ptr(stream)
        table, K, _ = layer_table(lv, spec.kernel)
        cin, cout = spec.in_channels, spec.out_channels
        dev = dy_rows.device
        dz = torch.zeros((lv.cap, cout), dtype=torch.float32, device=dev)
        _lib.call("fpvs_act_backward", _lib.ptr(dy_rows.contiguous()), dy_rows.shape[1], _lib.ptr(cache.y_rows),
                  _lib.F32, cache.y_rows.shape[1], _lib.ptr(lv.n), lv.cap, cout, _lib.ACT[spec.activation], _lib.ptr(dz),
                  cout, s)
        dw = torch.zeros((K * cin, cout), dtype=torch.float32, device=dev)
        db = torch.zeros(cout, dtype=torch.float32, device=dev)
        ws = torch.empty(_lib.size("fpvs_wgrad_workspace_size", K, cin, cout, lv.cap), dtype=torch.uint8, device=dev)
        _lib.call("fpvs_spconv_wgrad_simt", _lib.ptr(cache.x_rows), cache.x_rows.shape[1], _lib.F32, _lib.ptr(dz), cout,
                  _lib.ptr(table), K, _lib.ptr(lv.n), lv.cap, cin, cout, _lib.ptr(dw), _lib.ptr(db), _lib.ptr(ws),
                  ws.numel(), s)
        dx = None
        if need_dx:
            dx = torch.zeros((lv.cap, cin), dtype=torch.float32, device=dev)
            _lib.call("fpvs_spconv_dgrad_simt", _lib.ptr(dz), cout, _lib.ptr(table), K, _lib.ptr(lv.n), lv.cap,
                      _lib.ptr(self.w.contiguous()), cin, cout, None, _lib.F32, 0, _lib.ptr(dx), cin, s)
        return dx, dw, db


@dataclass
class Conv3dCache:
    """What Conv3d.backward needs (the reference keeps (cols, z, y, shape),
    neural.py:219): the active set, the input rows and the output rows."""
    level: object
    x_rows: object
    y_rows: object
    shape: tuple
    host: bool


def conv3d_forward(x, layer: Conv3d):
    """neural.py:252-253."""
    return layer.forward(x)


def conv3d_backward(layer: Conv3d, dy, cache):
    """neural.py:256-257."""
    return layer.backward(dy, cache)


def _dense_in(x, channels: int):
    """(B, X, Y, Z, C) numpy / tensor -> contiguous f32 CUDA tensor, shape-checked as neural.py:203-205."""
    torch = _torch()
    xt = x.to("cuda", torch.float32) if isinstance(x, torch.Tensor) else \
        torch.as_tensor(np.asarray(x, dtype=np.float32)).cuda()
    if xt.dim() != 5 or xt.shape[4] != channels:
        raise ValueError(f"expected (B, D, H, W, {channels}) input, got {tuple(xt.shape)}")
    return xt.contiguous()


def dense_level(xt) -> sp.Level:
    """Level of a dense (B, X, Y, Z, C) tensor: active = any nonzero channel, C-order rows, 3^3 map."""
    torch = _torch()
    B, X, Y, Z, _ = xt.shape
    lv = sp.new_level(B, (X, Y, Z))
    lv.active.copy_((xt != 0).any(-1).reshape(-1).to(torch.uint8))
    sp.compact(lv)
    sp.build_subm(lv)
    return lv


def _row_index(lv: sp.Level):
    c = lv.coords[:lv.count()].long()
    X, Y, Z = lv.dims
    return ((c[:, 0] * X + c[:, 1]) * Y + c[:, 2]) * Z + c[:, 3]


def dense_to_rows(xt, lv: sp.Level):
    """Active rows (cap, C) f32 of a dense (B, X, Y, Z, C) tensor (zero past the count)."""
    torch = _torch()
    C = xt.shape[-1]
    rows = torch.zeros((lv.cap, C), dtype=torch.float32, device=xt.device)
    idx = _row_index(lv)
    rows[:len(idx)] = xt.reshape(-1, C)[idx].to(torch.float32)
    return rows


def rows_to_dense(rows, lv: sp.Level, C: int):
    """Scatter active rows back to a dense (B, X, Y, Z, C) f32 tensor (0 at inactive cells)."""
    torch = _torch()
    X, Y, Z = lv.dims
    out = torch.zeros((lv.B * X * Y * Z, C), dtype=torch.float32, device=rows.device)
    idx = _row_index(lv)
    out[idx] = rows[:len(idx), :C].to(torch.float32)
    return out.reshape(lv.B, X, Y, Z, C)


def packed_cache(layer, bn: int = 0, stream=None):
    """The layer's bf16 weight image for tile width ``bn`` (built once per bn)."""
    if layer._packed is None:
        layer._packed = {}
    if bn not in layer._packed:
        layer._packed[bn] = pack_tc(layer.w, layer.taps, layer.spec.in_channels, layer.spec.out_channels, bn, stream)
    return layer._packed[bn]


def repack_all(layers, stream=None):
    """Refresh every cached bf16 weight image of ``layers`` from their (updated)
    fp32 weights in ONE launch (fpvs_pack_weights_tc_multi) — the training
    step's re-pack after each optimizer update; images of other kinds are
    dropped and rebuilt lazily."""
    import ctypes as C
    jobs = []
    for L in layers:
        cache = getattr(L, "_packed", None)
        if not cache:
            continue
        for key in list(cache):
            cin, cout = L.spec.in_channels, L.spec.out_channels
            if isinstance(key, int):
                jobs.append((L.w, L.taps, cin, cout, key, 0, cache[key]))
            elif isinstance(key, tuple) and key[0] == "dgrad":
                jobs.append((L.w, L.taps, cin, cout, key[1], 1, cache[key]))
            else:
                del cache[key]
    for i in range(0, len(jobs), 32):
        part = jobs[i:i + 32]
        arr = (_lib.PackJob * len(part))()
        for e, (w, taps, cin, cout, bn, dg, out) in zip(arr, part):
            e.w, e.K, e.cin, e.cout, e.bn, e.dgrad, e.packed = _lib.ptr(w), taps, cin, cout, bn, dg, _lib.ptr(out)
        _lib.call("fpvs_pack_weights_tc_multi", C.addressof(arr), len(part), _lib.stream_ptr(stream))


def packed_upblocks_cache(layer, bn: int = 0, stream=None):
    """The k2s2 up layer's weights as one Cin x 8 Cout matrix (column block j =
    parity class j's slice, fpvs_spconv_tc_upblocks) and its bias tiled 8
    times; built once per update."""
    if layer._packed is None:
        layer._packed = {}
    key = ("upblocks", bn)
    if key not in layer._packed:
        cin, cout = layer.spec.in_channels, layer.spec.out_channels
        if layer.taps != 8:
            raise ValueError(f"up blocks need a k = 2 layer, got {layer.taps} taps")
        w8 = layer.w.view(8, cin, cout).permute(1, 0, 2).reshape(cin, 8 * cout).contiguous()
        layer._packed[key] = (pack_tc(w8, 1, cin, 8 * cout, bn, stream), layer.b.repeat(8).contiguous())
    return layer._packed[key]


def packed_dgrad_cache(layer, bn: int = 0, stream=None):
    """The layer's dgrad weight image (mirrored offsets, per-offset Wᵀ), built once per update."""
    if layer._packed is None:
        layer._packed = {}
    key = ("dgrad", bn)
    if key not in layer._packed:
        torch = _torch()
        cin, cout = layer.spec.in_channels, layer.spec.out_channels
        nbytes = _lib.size("fpvs_pack_weights_tc_size", layer.taps, cout, cin, bn)
        if nbytes == 0:
            raise ValueError(f"no tensor-core dgrad packing for taps={layer.taps}, Cin={cin}, Cout={cout}")
        out = torch.empty(nbytes, dtype=torch.uint8, device=layer.w.device)
        _lib.call("fpvs_pack_weights_tc_dgrad", _lib.ptr(layer.w.contiguous()), layer.taps, cin, cout, bn,
                  _lib.ptr(out), _lib.stream_ptr(stream))
        layer._packed[key] = out
    return layer._packed[key]


def pack_tc(w, taps: int, cin: int, cout: int, bn: int = 0, stream=None):
    torch = _torch()
    nbytes = _lib.size("fpvs_pack_weights_tc_size", taps, cin, cout, bn)
    if nbytes == 0:
        raise ValueError(f"no tensor-core packing for taps={taps}, Cin={cin}, Cout={cout}, bn={bn}")
    out = torch.empty(nbytes, dtype=torch.uint8, device=w.device)
    _lib.call("fpvs_pack_weights_tc", _lib.ptr(w.contiguous()), taps, cin, cout, bn, _lib.ptr(out),
              _lib.stream_ptr(stream))
    return out


def pick_bn(cout: int, rows: int, sms: int = 148) -> int:
    """Output-tile width: split N until the layer has >= one wave of 128-row tiles."""
    bn = 32 if cout <= 32 else 64 if cout <= 64 else 128 if cout <= 128 else 256
    mtiles = max(1, (rows + 127) // 128)
    # splitting N re-gathers A once per column block; measured on B200 it only
    # pays when the layer has well under half a wave of row tiles
    while bn > 64 and mtiles * ((cout + bn - 1) // bn) < sms // 2:
        bn //= 2
    return bn


def layer_table(lv: sp.Level, k: int):
    """(table, K, tile masks) a kernel-k submanifold conv reads on level ``lv``.

    k = 3 is the level's own table; other odd k get a k^3-tap table in
    ``lv.extra`` that :func:`build_layer_tables` (re)fills after every map build.
    """
    if k == 1:
        return None, 1, None
    if k == 3:
        return lv.nbr, 27, lv.nbr_masks
    key = ("nbr", k)
    t = lv.extra.get(key)
    if t is None:
        torch = _torch()
        t = torch.empty((lv.cap, k ** 3), dtype=torch.int32, device=lv.coords.device)
        lv.extra[key] = t
    return t, k ** 3, None


def build_layer_tables(lv: sp.Level, kernels, stream=None):
    """Fill the k^3-tap tables (k not in {1, 3}) of ``kernels`` from the level's
    coordinates and index volume (one fpvs_kmap_subm_k launch per distinct k)."""
    X, Y, Z = lv.dims
    for k in sorted(set(kernels)):
        if k in (1, 3):
            continue
        t, _, _ = layer_table(lv, k)
        _lib.call("fpvs_kmap_subm_k", _lib.ptr(lv.coords), _lib.ptr(lv.n), lv.cap, _lib.ptr(lv.index_vol), lv.B, X, Y,
                  Z, k, _lib.ptr(t), _lib.stream_ptr(stream))


def tc_ok(K: int, cin: int, cout: int, act: str = "relu") -> bool:
    """Shapes the tcgen05 gather-GEMM (fpvs_spconv_tc) takes; others run on the
    SIMT kernel with bf16 operands."""
    return K <= 27 and cin % 8 == 0 and cout % 32 == 0 and cout <= 1024 and act in ("relu", "none")


def halo_ok(K: int, cin: int, cout: int, dtype=None) -> bool:
    """Shapes the halo-cached tensor-core conv (fpvs_spconv_halo) takes."""
    return K == 27 and (cin % 64 == 0 or cin == 32) and cout % 32 == 0 and cout <= 1024


def brick_ok(K: int, cin: int, cout: int, dtype=None) -> bool:
    """Shapes the dense-brick conv takes (fpvs_spconv_brick)."""
    torch = _torch()
    if dtype is not None and dtype != torch.bfloat16:
        return False
    return K == 27 and cin % 64 == 0 and cout % 64 == 0 and cout <= 1024


def run_conv(layer: Conv3d, x, ldx: int, table, K: int, n, cap: int, y, ldy: int, col_off: int = 0,
             precision: str = "fp32", act: str | None = None, stream=None, bn: int = 0, masks=None,
             halo=None, halo_tabs=None, out_rows=None, settled: bool = False, done_out=None, done_in=None,
             done_n=None, brick=None):
    """One sparse conv launch: y[:, col_off:col_off+Cout] = act(gather-GEMM(x, table) + b).

    ``masks`` are the table's per-tile offset masks (sparse.tile_masks); the
    tensor-core path computes them here when not given.  ``halo`` =
    (bn, split, workspace) with ``halo_tabs`` (sparse.build_halo) selects the
    halo-cached kernel for 27-tap layers with 64-multiple channels.
    ``out_rows`` (bf16 only) maps tile row i to output row out_rows[i]
    (-1 = skip): the parity-sorted up conv (sparse.UpSorter).  ``settled``:
    the tables and tile masks were written two or more launches earlier (the
    halo conv may then decode its units before its programmatic-launch wait,
    FPVS_TABLES_SETTLED).  ``done_out`` / ``done_in``: per-tile dataflow flags
    between two halo convs of one level (fpvs_spconv_halo_flow); the plain
    gather-GEMM takes ``done_in`` with ``done_n``, the producer level's row
    count (fpvs_spconv_tc_flow).  ``brick`` = (bn, split, workspace, level):
    the dense-brick kernel for a well-filled level (fpvs_spconv_brick; reads
    the level's index volume instead of ``table``).
    """
    torch = _torch()
    spec = layer.spec
    a = _lib.ACT[act or spec.activation]
    s = _lib.stream_ptr(stream)
    if precision == "bf16" and out_rows is None and not tc_ok(K, spec.in_channels, spec.out_channels,
                                                              act or spec.activation):
        precision = "simt"  # e.g. k = 5 (125 taps): SIMT FFMA on the bf16 rows
    if precision == "bf16":
        if table is not None and masks is None:
            masks = sp.tile_masks(table, K, n, cap, stream=stream)
        if brick is not None and brick_ok(K, spec.in_channels, spec.out_channels, x.dtype):
            bbn, bsplit, ws, lv = brick
            X, Y, Z = lv.dims
            _lib.call("fpvs_spconv_brick", _lib.ptr(x), ldx, x.shape[0], _lib.ptr(lv.index_vol), lv.B, X, Y, Z,
                      _lib.ptr(layer.packed(bbn, stream)), bbn, bsplit, _lib.ptr(layer.b), spec.in_channels,
                      spec.out_channels, a | (_lib.TABLES_SETTLED if settled else 0), _lib.ptr(y), ldy, col_off, _lib.ptr(ws), 0 if ws is None else ws.numel(),
                      s)
            return
        if halo is not None and halo_ok(K, spec.in_channels, spec.out_channels, x.dtype):
            hbn, split, ws = halo
            args = [_lib.ptr(x), ldx, x.shape[0], _lib.ptr(table), _lib.ptr(halo_tabs["lnbr"]),
                    _lib.ptr(halo_tabs["rows"]), _lib.ptr(halo_tabs["n"]), _lib.ptr(masks), _lib.ptr(n), cap,
                    _lib.ptr(layer.packed(hbn, stream)), hbn, split, _lib.ptr(layer.b), spec.in_channels,
                    spec.out_channels, a | (_lib.TABLES_SETTLED if settled else 0), _lib.ptr(y), ldy, col_off,
                    _lib.ptr(ws), ws.numel()]
            if done_out is not None or done_in is not None:
                _lib.call("fpvs_spconv_halo_flow", *args, _lib.ptr(done_out), _lib.ptr(done_in), s)
            else:
                _lib.call("fpvs_spconv_halo", *args, s)
            return
        if out_rows is not None:
            _lib.call("fpvs_spconv_tc_scatter", _lib.ptr(x), ldx, x.shape[0], _lib.ptr(table), K, _lib.ptr(masks),
                      _lib.ptr(n), cap, _lib.ptr(out_rows), _lib.ptr(layer.packed(bn, stream)), bn, _lib.ptr(layer.b),
                      spec.in_channels, spec.out_channels, a, _lib.ptr(y), ldy, col_off, s)
            return
        targs = [_lib.ptr(x), ldx, x.shape[0], _lib.ptr(table), K, _lib.ptr(masks), _lib.ptr(n), cap,
                 _lib.ptr(layer.packed(bn, stream)), bn, _lib.ptr(layer.b), spec.in_channels, spec.out_channels, a,
                 _lib.ptr(y), ldy, col_off]
        if done_in is not None:
            if done_n is None:
                raise ValueError("a gather-GEMM dataflow consumer needs the producer's row count (done_n)")
            _lib.call("fpvs_spconv_tc_flow", *targs, _lib.ptr(done_in), _lib.ptr(done_n), s)
        else:
            _lib.call("fpvs_spconv_tc", *targs, s)
    else:
        idt = _lib.BF16 if x.dtype == torch.bfloat16 else _lib.F32
        odt = _lib.BF16 if y.dtype == torch.bfloat16 else _lib.F32
        _lib.call("fpvs_spconv_simt", _lib.ptr(x), ldx, idt, _lib.ptr(table), K, _lib.ptr(n), cap,
                  _lib.ptr(layer.w), _lib.ptr(layer.b), spec.in_channels, spec.out_channels, a, _lib.ptr(y), ldy,
                  col_off, odt, s)


def run_head(layer: Conv3d, x, ldx: int, lv: sp.Level, d: int, grid_dims, tau: float, out_bits=None,
             probs=None, logits=None, precision: str = "fp32", stream=None):
    """Head + sigmoid + [p >= tau] + deinterleave bit-pack (neural.py:513-526).

    A 1x1x1 head is one fused kernel; a k^3 head (the reference default,
    neural.py:94-99) runs as a conv with no activation into f32 logits rows
    (SIMT, exact fp32 accumulation) followed by fpvs_head_rows."""
    torch = _torch()
    nx, ny, nz = grid_dims
    s = _lib.stream_ptr(stream)
    spec = layer.spec
    if spec.kernel != 1:
        d3 = d ** 3
        table, K, _ = layer_table(lv, spec.kernel)
        lg = logits
        if lg is None:
            lg = lv.extra.get("head_logits")
            if lg is None or lg.shape[1] != d3:
                lg = torch.empty((lv.cap, d3), dtype=torch.float32, device=x.device)
                lv.extra["head_logits"] = lg
        idt = _lib.BF16 if x.dtype == torch.bfloat16 else _lib.F32
        _lib.call("fpvs_spconv_simt", _lib.ptr(x), ldx, idt, _lib.ptr(table), K, _lib.ptr(lv.n), lv.cap,
                  _lib.ptr(layer.w), _lib.ptr(layer.b), spec.in_channels, d3, _lib.ACT["none"], _lib.ptr(lg),
                  lg.shape[1], 0, _lib.F32, s)
        _lib.call("fpvs_head_rows", _lib.ptr(lg), lg.shape[1], _lib.ptr(lv.coords), _lib.ptr(lv.n), lv.cap, d, lv.B,
                  nx, ny, nz, float(tau), _lib.ptr(out_bits), _lib.ptr(probs), s)
        return
    if precision == "bf16":
        _lib.call("fpvs_head_tc", _lib.ptr(x), ldx, x.shape[0], _lib.ptr(lv.coords), _lib.ptr(lv.n), lv.cap,
                  _lib.ptr(layer.packed(0, stream)), _lib.ptr(layer.b), spec.in_channels, d, lv.B, nx, ny, nz,
                  float(tau), _lib.ptr(out_bits), _lib.ptr(probs), _lib.ptr(logits), s)
    else:
        idt = _lib.BF16 if x.dtype == torch.bfloat16 else _lib.F32
        _lib.call("fpvs_head_simt", _lib.ptr(x), ldx, idt, _lib.ptr(lv.coords), _lib.ptr(lv.n), lv.cap,
                  _lib.ptr(layer.w), _lib.ptr(layer.b), spec.in_channels, d, lv.B, nx, ny, nz, float(tau),
                  _lib.ptr(out_bits), _lib.ptr(probs), _lib.ptr(logits), s)


# ---------------------------------------------------------------------------
# network
# ---------------------------------------------------------------------------

class PvsNet:
    """Stack of submanifold convs mapping interleaved cells to probabilities (neural.py:260-346)."""

    OUTPUT_GAIN = 3.0

    def __init__(self, cfg: ModelConfig, rng: np.random.Generator | None = None, device: str = "cuda",
                 precision: str = "fp32"):
        _lib.require_cuda()
        if precision not in ("fp32", "bf16"):
            raise ValueError(f"unknown precision {precision!r}")
        self.cfg = cfg
        self.precision = precision
        self.layers = [Conv3d(spec, rng, cfg.init, device) for spec in cfg.layers]
        if cfg.init == "identity" and rng is not None:
            for layer in self.layers[:-1]:
                layer.seed_identity(rng, 1.0)
            self.layers[-1].seed_identity(rng, self.OUTPUT_GAIN)
            self.layers[-1].b.fill_(-self.OUTPUT_GAIN / 2.0)

    # -- device path ---------------------------------------------------------
    def kernels(self):
        return [L.spec.kernel for L in self.layers]

    def forward_rows(self, feats, lv: sp.Level, grid_dims, tau: float = 0.5, out_bits=None, probs=None,
                     logits=None, keep: bool = False, stream=None):
        """Run the chain on active-cell rows; the head writes bits / probs / logits.

        Returns the list of per-layer activations when ``keep`` (training).
        """
        torch = _torch()
        d = self.cfg.d
        bf16 = self.precision == "bf16"
        dt = torch.bfloat16 if bf16 else torch.float32
        build_layer_tables(lv, self.kernels(), stream)
        x = feats
        acts = [x]
        for layer in self.layers[:-1]:
            y = torch.empty((lv.cap, layer.spec.out_channels), dtype=dt, device=x.device)
            table, K, masks = layer_table(lv, layer.spec.kernel)
            run_conv(layer, x, x.shape[1], table, K, lv.n, lv.cap, y, y.shape[1], 0, self.precision, stream=stream,
                     masks=masks)
            x = y
            acts.append(x)
        run_head(self.layers[-1], x, x.shape[1], lv, d, grid_dims, tau, out_bits, probs, logits,
                 self.precision, stream)
        return acts if keep else None

    def predict_bits(self, bits, B: int, grid_dims, tau: float = 0.5, stream=None, level: sp.Level | None = None):
        """Packed PVS bits of B packed grids, all on the device (no host sync)."""
        torch = _torch()
        d = self.cfg.d
        lv = level or sp.level_from_bits(bits, B, grid_dims, d, stream=stream)
        dt = torch.bfloat16 if self.precision == "bf16" else torch.float32
        feats = sp.gather_features(bits, lv, grid_dims, d, dt, stream=stream)
        nx, ny, nz = grid_dims
        out = torch.zeros(B * nx * ny * nz // 8, dtype=torch.uint8, device=bits.device)
        self.forward_rows(feats, lv, grid_dims, tau, out_bits=out, stream=stream)
        return out

    # -- reference-shaped dense API (neural.py:260-297) ------------------------
    def _dense_level(self, x):
        xt = _dense_in(x, self.cfg.layers[0].in_channels)
        return xt, dense_level(xt)

    def forward(self, x):
        """(B, X, Y, Z, d^3) -> probabilities of the same shape; inactive cells -> 0."""
        torch = _torch()
        host = not isinstance(x, torch.Tensor)
        xt, lv = self._dense_level(x)
        B, X, Y, Z, C = xt.shape
        feats = dense_to_rows(xt, lv)
        if self.precision == "bf16":
            feats = feats.to(torch.bfloat16)
        d3 = self.cfg.layers[-1].out_channels
        probs = torch.zeros((lv.cap, d3), dtype=torch.float32, device="cuda")
        grid_dims = (X * self.cfg.d, Y * self.cfg.d, Z * self.cfg.d)
        self.forward_rows(feats, lv, grid_dims, 0.5, probs=probs)
        out = rows_to_dense(probs, lv, d3)
        return out.cpu().numpy().astype(np.float64) if host else out

    def forward_cached(self, x):
        """(probabilities, per-layer caches) as neural.py:263-268; fp32 on the device."""
        torch = _torch()
        host = not isinstance(x, torch.Tensor)
        xt, lv = self._dense_level(x)
        rows = dense_to_rows(xt, lv)
        caches = []
        for layer in self.layers:
            y_rows = layer.forward_rows_f32(rows, lv)
            caches.append(Conv3dCache(lv, rows, y_rows, tuple(xt.shape[:4]) + (layer.spec.out_channels,), host))
            rows = y_rows
        out = rows_to_dense(rows, lv, self.layers[-1].spec.out_channels)
        return (out.cpu().numpy().astype(np.float64) if host else out), caches

    def backward(self, dy, caches):
        """Per-layer (dw, db) gradients plus the input gradient (neural.py:270-276)."""
        torch = _torch()
        if not caches:
            raise ValueError("backward requires the forward caches")
        host = not isinstance(dy, torch.Tensor)
        lv = caches[-1].level
        g = dense_to_rows(_dense_in(dy, self.layers[-1].spec.out_channels), lv)
        grads = [None] * len(self.layers)
        for i in reversed(range(len(self.layers))):
            g, dw, db = self.layers[i].backward_rows(g, caches[i])
            grads[i] = (dw, db)
        dx = rows_to_dense(g, lv, self.layers[0].spec.in_channels)
        if host:
            grads = [(dw.cpu().numpy().astype(np.float64), db.cpu().numpy().astype(np.float64)) for dw, db in grads]
            dx = dx.cpu().numpy().astype(np.float64)
        return grads, dx

    def sgd_step(self, grads, lr: float):
        """w -= lr dw, b -= lr db per layer (neural.py:278-281), fpvs_sgd_step on the device."""
        torch = _torch()
        for layer, (dw, db) in zip(self.layers, grads):
            for param, grad in ((layer.w, dw), (layer.b, db)):
                gt = torch.as_tensor(grad if isinstance(grad, torch.Tensor) else np.asarray(grad, dtype=np.float32),
                                     dtype=torch.float32).to(param.device).reshape(param.shape).contiguous()
                _lib.call("fpvs_sgd_step", _lib.ptr(param), _lib.ptr(gt), param.numel(), float(lr),
                          _lib.stream_ptr())
            layer.invalidate()

    def parameters(self):
        out = []
        for layer in self.layers:
            out += [layer.w, layer.b]
        return out

    def invalidate(self):
        for layer in self.layers:
            layer.invalidate()

    # -- checkpoint format (neural.py:299-346) -------------------------------
    def save(self, path):
        lines = [f"d={self.cfg.d}"]
        for spec in self.cfg.layers:
            lines.append(f"layer={spec.kernel}:{spec.in_channels}:{spec.out_channels}:{spec.activation}")
        text = "\n".join(lines).encode()
        with open(path, "wb") as fh:
            fh.write(FPVW_MAGIC + struct.pack("<II", FPVW_VERSION, len(text)))
            fh.write(text)
            for layer in self.layers:
                fh.write(layer.w.detach().cpu().numpy().astype("<f4").tobytes())
                fh.write(layer.b.detach().cpu().numpy().astype("<f4").tobytes())

    @classmethod
    def load(cls, path, precision: str = "fp32") -> "PvsNet":
        d, specs, arrays = read_fpvw(path)
        net = cls(ModelConfig(d, specs), precision=precision)
        for layer, (w, b) in zip(net.layers, arrays):
            layer.set_weights(w, b)
        return net


def read_fpvw(path):
    """Parse an FPVW checkpoint: (d, [ConvSpec], [(w (k^3 Cin, Cout) f32, b f32)]) (neural.py:316-346)."""
    raw = Path(path).read_bytes()
    if raw[:4] != FPVW_MAGIC:
        raise ValueError(f"{path}: not an FPVW checkpoint")
    version, textlen = struct.unpack_from("<II", raw, 4)
    if version != FPVW_VERSION:
        raise ValueError(f"{path}: unsupported FPVW version {version}")
    text = raw[12:12 + textlen].decode()
    d, specs = None, []
    for line in text.splitlines():
        key, val = line.split("=", 1)
        if key == "d":
            d = int(val)
        elif key == "layer":
            k, cin, cout, act = val.split(":")
            specs.append(ConvSpec(int(k), int(cin), int(cout), act))
    off = 12 + textlen
    arrays = []
    for s in specs:
        nw = s.kernel ** 3 * s.in_channels * s.out_channels
        w = np.frombuffer(raw, "<f4", nw, off).reshape(s.kernel ** 3 * s.in_channels, s.out_channels).copy()
        off += 4 * nw
        b = np.frombuffer(raw, "<f4", s.out_channels, off).copy()
        off += 4 * s.out_channels
        arrays.append((w, b))
    return d, specs, arrays


# ---------------------------------------------------------------------------
# losses (neural.py:353-399), evaluated on the GPU
# ---------------------------------------------------------------------------

def dice_loss(pred, gt, alpha: float):
    """Weighted Dice 1 - 2TP/(2TP + alpha FP + (1-alpha) FN); returns (value, grad)."""
    p, g = _as_cuda64(pred), _as_cuda64(gt)
    if p.shape != g.shape:
        raise ValueError("prediction and ground truth shapes differ")
    tp = (p * g).sum()
    fp = p.sum() - tp
    fn = g.sum() - tp
    num = 2.0 * tp
    den = 2.0 * tp + alpha * fp + (1.0 - alpha) * fn
    if float(den) == 0.0:
        return 0.0, _like(pred, np.zeros(tuple(p.shape)))
    dden = 2.0 * g + alpha * (1.0 - g) - (1.0 - alpha) * g
    grad = -(2.0 * g * den - num * dden) / (den * den)
    return float((den - num) / den), _like(pred, grad)


def rvl_loss(pred, gt):
    """Repulsive visibility loss (1 - TP/GTP) + FP/GTP; returns (value, grad)."""
    p, g = _as_cuda64(pred), _as_cuda64(gt)
    if p.shape != g.shape:
        raise ValueError("prediction and ground truth shapes differ")
    gtp = float(g.sum())
    if gtp == 0.0:
        return 0.0, _like(pred, np.zeros(tuple(p.shape)))
    tp = float((p * g).sum())
    fp = float(p.sum()) - tp
    return (1.0 - tp / gtp) + fp / gtp, _like(pred, (1.0 - 2.0 * g) / gtp)


def combined_loss(pred, gt, cfg: TrainConfig):
    dv, dg = dice_loss(pred, gt, cfg.alpha)
    rv, rg = rvl_loss(pred, gt)
    return cfg.lam * dv + (1.0 - cfg.lam) * rv, cfg.lam * dg + (1.0 - cfg.lam) * rg


def _like(ref, val):
    """Gradient in the caller's form: a tensor on the caller's device for tensor
    input, a float64 numpy array for numpy input (neural.py returns np arrays)."""
    torch = _torch()
    if isinstance(ref, torch.Tensor):
        return (val if isinstance(val, torch.Tensor) else torch.as_tensor(val)).to(ref.device)
    return val.cpu().numpy() if isinstance(val, torch.Tensor) else np.asarray(val)


# ---------------------------------------------------------------------------
# inference entry (neural.py:513-526)
# ---------------------------------------------------------------------------

def predict_pvs(grid: FroxelGrid, net, tau: float = 0.5) -> FroxelGrid:
    """Interleave, run the network, deinterleave with threshold tau — one device pass."""
    torch = _torch()
    if isinstance(net, (str, Path)):
        net = PvsNet.load(net)
    d = net.cfg.d
    if any(dim % d for dim in grid.dims):
        raise ValueError(f"grid dims {grid.dims} not divisible by interleave factor {d}")
    if net.cfg.layers[0].in_channels != d ** 3:
        raise ValueError("grid/channel mismatch against the checkpoint")
    bits = torch.from_numpy(grid.bits).cuda()
    out = net.predict_bits(bits, 1, grid.dims, tau)
    res = FroxelGrid(grid.dims, role="predicted_pvs", bits=out.cpu().numpy())
    res.supersample = grid.supersample
    return res


# ---------------------------------------------------------------------------
# training entry points (neural.py:405-510), implemented in .train
# ---------------------------------------------------------------------------

def train(pairs, mcfg: ModelConfig, tcfg: TrainConfig, eval_pairs=None, target_fnr=None, target_fpr=None,
          checkpoint_path=None, log_path=None, verbose: bool = False, precision: str = "fp32"):
    """Drop-in ``train`` (neural.py:442-510); see paper_2509_24677_b200.train.train."""
    from .train import train as _train
    return _train(pairs, mcfg, tcfg, eval_pairs, target_fnr, target_fpr, checkpoint_path, log_path, verbose,
                  precision)


def _tensor_pairs(pairs, d: int):
    """Stacked interleaved (geometry, gt) tensors of FroxelGrid pairs (neural.py:415-420), float64 numpy."""
    from .interleave import interleave
    xs, ys = [], []
    for geo, gt in pairs:
        xs.append(interleave(geo, d).values)
        ys.append(interleave(gt, d).values)
    return np.stack(xs), np.stack(ys)


def _epoch_rates(tp, fp, fn, gtp):
    """(FNR, FPR) = (FN / GTP, FP / GTP), (0, 0) without positives (neural.py:423-426)."""
    if gtp == 0:
        return 0.0, 0.0
    return fn / gtp, fp / gtp


def evaluate_pairs(net: PvsNet, x, y, tau: float, batch: int = 8):
    """Hard FNR/FPR of thresholded predictions over a stacked pair set
    (neural.py:429-439): pred = p >= tau over every cell (inactive cells have
    p = 0), gt = y > 0.5; counted on the device, ``batch`` samples per pass."""
    torch = _torch()
    n = len(x)
    tot = torch.zeros(4, dtype=torch.int64, device="cuda")
    for i in range(0, n, batch):
        xs = x[i:i + batch]
        probs = net.forward(xs if isinstance(xs, torch.Tensor) else torch.as_tensor(np.asarray(xs, np.float32)).cuda())
        ys = y[i:i + batch]
        gt = (ys.cuda() if isinstance(ys, torch.Tensor) else torch.as_tensor(np.asarray(ys, np.float32)).cuda()) > 0.5
        pred = probs >= tau
        tot += torch.stack([(pred & gt).sum(), (pred & ~gt).sum(), (~pred & gt).sum(), gt.sum()])
    tp, fp, fn, gtp = (int(v) for v in tot.cpu())
    return _epoch_rates(tp, fp, fn, gtp)


def evaluate_grid_pairs(net: PvsNet, pairs, tau: float):
    """Hard FNR/FPR over (geometry, gt) FroxelGrid pairs on packed bits (fpvs_bits_confusion)."""
    from .train import evaluate_grid_pairs as _ev
    return _ev(net, pairs, tau)


def load_pairs(manifest_path) -> list:
    """(geometry, gt) pairs of a dataset manifest (neural.py:405-411)."""
    from .train import load_pairs as _lp
    return _lp(manifest_path)
