"""Training hot path (SURVEY.md §8(a) rows BW, LOSS, TR, EVAL, CKPT; BASELINE config 5).

``train`` keeps the reference's signature and loop structure
(pkg/src/froxelpvs/neural.py:442-510): PCG64(seed) drives the initial weights
and the per-epoch permutation, the loss is the per-sample combined loss
averaged over the batch (neural.py:472-477), a non-finite loss raises
``TrainingDiverged``, the update is SGD at lr * (1 - decay)^step
(neural.py:481) — or AdamW with fp32 master weights when
``TrainConfig.optimizer == "adamw"`` (config 5) — and the history holds the
epoch's mean loss and hard FNR/FPR at ``tau``.

A step runs entirely on the device through the C ABI:

  maps        fpvs_levels_from_bits (active cells, neighbour table, features,
              clears the prediction grid)
  forward     per layer fpvs_spconv_tc (bf16) / fpvs_spconv_simt (fp32), every
              activation kept (the cache of neural.py:263-275)
  head        fused 1x1x1 conv + sigmoid: probabilities + thresholded bits
  loss        fpvs_loss_counts + fpvs_loss_grad: per-sample (TP, sum p, GTP)
              in f64, dL/dlogit = G_g * p (1 - p) / B (neural.py:353-399)
  counts      fpvs_bits_confusion: hard TP/FP/FN/GTP from packed bits
  backward    per layer fpvs_spconv_wgrad_simt (dW, db into ONE flat fp32
              gradient) and fpvs_spconv_dgrad_simt (mirrored-offset gather
              with Wᵀ, relu' = z > 0 from the kept activation)
  exchange    world > 1: one all-reduce of the flat gradient (NCCL over NVLink)
  update      fpvs_sgd_step / fpvs_adamw_step on the flat fp32 parameters

Data parallelism: each rank takes a strided share of every global batch; the
local mean gradient is weighted by B_local / B_global and summed across ranks,
which equals the reference's global batch mean for any split.

Submanifold semantics: inactive cells predict p = 0,
so they add nothing to TP / FP and their labels count only in GTP (labels are a
subset of the occupancy, row LBL).
"""

from __future__ import annotations

import os
from pathlib import Path

import numpy as np

from . import _lib
from . import sparse as sp
from .froxel import FroxelGrid
from .neural import (ModelConfig, PvsNet, TrainConfig, TrainingDiverged, build_layer_tables, layer_table,
                     packed_dgrad_cache, run_conv, run_head, halo_ok, repack_all)


def _torch():
    import torch
    return torch


def _dist():
    import torch.distributed as dist
    return dist if dist.is_available() and dist.is_initialized() else None


def shard(indices, rank: int, world: int):
    """Rank ``rank``'s strided share of one global batch (may be empty)."""
    return list(indices)[rank::world]


def allreduce_weighted(flat, weight: float):
    """flat <- sum over ranks of weight_r * flat_r (one all-reduce; identity at world 1).

    With weight_r = B_r / B_global and flat_r the rank's local mean gradient,
    the result is the global batch mean on every rank.
    """
    dist = _dist()
    if weight != 1.0:
        flat.mul_(weight)
    if dist is not None and dist.get_world_size() > 1:
        dist.all_reduce(flat, op=dist.ReduceOp.SUM)
    return flat


def use_halo_wgrad() -> bool:
    """FPVS_HALO_WGRAD=0 keeps every layer on the gathering wgrad (A/B checks)."""
    import os
    return os.environ.get("FPVS_HALO_WGRAD", "1") != "0"


class TrainStep:
    """All device buffers of one (B, grid) training step; ``run`` only launches kernels.

    The network's weights become views into one flat fp32 buffer (the master
    copy the optimizer updates); the gradient has the same flat layout.
    """

    def __init__(self, net: PvsNet, B: int, grid_dims, tcfg: TrainConfig, device="cuda"):
        torch = _torch()
        self.net, self.B, self.grid_dims, self.tcfg = net, B, tuple(grid_dims), tcfg
        d = net.cfg.d
        nx, ny, nz = self.grid_dims
        if nx % 8 or nx % d or ny % d or nz % d:
            raise ValueError(f"grid dims {self.grid_dims} not divisible by interleave factor {d} (N_x by 8)")
        self.grid_bytes = nx * ny * nz // 8
        self.lv = sp.new_level(B, (nx // d, ny // d, nz // d), device=device)
        bf16 = net.precision == "bf16"
        tc_bw = bf16 and self._tc_backward_ok()
        # 27-tap layers with Cin = 32 take the halo-cached wgrad (wgrad_halo.cu)
        # and, where the shapes allow, the halo-cached forward: the level's halo
        # tables come out of the map build itself (K3), every step
        self.halo_wgrad = tc_bw and use_halo_wgrad() and any(self._halo_wgrad_ok(L) for L in net.layers)
        self.halo_fwd = bf16 and os.environ.get("FPVS_TRAIN_HALO_FWD", "1") != "0"
        want_halo = self.halo_wgrad or (self.halo_fwd and any(
            L.spec.kernel == 3 and halo_ok(27, L.spec.in_channels, L.spec.out_channels) for L in net.layers[:-1]))
        self.maps = sp.LevelMaps([self.lv], [], [], self.grid_dims, d, halo_levels=(0,) if want_halo else ())
        cap = self.lv.cap
        self.adt = torch.bfloat16 if bf16 else torch.float32
        self.x0 = torch.empty((cap, d ** 3), dtype=self.adt, device=device)
        self.acts = [torch.empty((cap, L.spec.out_channels), dtype=self.adt, device=device) for L in net.layers[:-1]]
        d3 = net.layers[-1].spec.out_channels
        self.probs = torch.empty((cap, d3), dtype=torch.float32, device=device)
        self.dlogits = torch.empty((cap, d3), dtype=torch.float32, device=device)
        widest = max(L.spec.in_channels for L in net.layers)
        self.dx = [torch.empty((cap, widest), dtype=torch.float32, device=device) for _ in range(2)]
        # bf16: the backward runs on tensor cores (tcgen05 dgrad / wgrad) with bf16 gradients
        self.tc_backward = tc_bw
        if self.tc_backward:
            self.dlog16 = torch.empty((cap, d3), dtype=torch.bfloat16, device=device)
            self.dz16 = [torch.empty((cap, widest), dtype=torch.bfloat16, device=device) for _ in range(2)]
            tws = max(_lib.size("fpvs_wgrad_tc_workspace_size", L.taps, L.spec.in_channels, L.spec.out_channels, cap)
                      for L in net.layers)
            self.wg_tc_ws = torch.empty(tws, dtype=torch.uint8, device=device)
            if self.halo_wgrad:
                self.wg_halo_ws = torch.empty(_lib.size("fpvs_wgrad_halo_workspace_size", cap), dtype=torch.uint8,
                                              device=device)
        self.halo_conv_ws = None
        if want_halo:
            def auto_bn(c):  # fpvs_spconv_halo's bn = 0 choice
                return 256 if c % 256 == 0 else 128 if c % 128 == 0 else 64 if c % 64 == 0 else 32
            need = max([_lib.size("fpvs_spconv_halo_workspace_size", cap, L.spec.out_channels,
                                  auto_bn(L.spec.out_channels), 1)
                        for L in net.layers[:-1] if L.spec.out_channels % 32 == 0] + [256])
            self.halo_conv_ws = torch.zeros(need, dtype=torch.uint8, device=device)
        self.pred_bits = torch.zeros(B * self.grid_bytes, dtype=torch.uint8, device=device)
        # flat master parameters and gradient
        sizes = [(L.w.numel(), L.b.numel()) for L in net.layers]
        total = sum(a + b for a, b in sizes)
        self.nparams = total
        self.params = torch.empty(total, dtype=torch.float32, device=device)
        # the exchange buffer: [flat gradient | loss + hard-count tail] (fpvs_exchange_pack)
        self.grads = torch.zeros(total + _lib.EXCHANGE_TAIL, dtype=torch.float32, device=device)
        self.tail = self.grads[total:]
        self.views = []
        o = 0
        for L, (nw, nb) in zip(net.layers, sizes):
            self.params[o:o + nw].copy_(L.w.reshape(-1))
            self.params[o + nw:o + nw + nb].copy_(L.b)
            L.w = self.params[o:o + nw].view(L.w.shape)
            L.b = self.params[o + nw:o + nw + nb]
            L.invalidate()
            self.views.append((self.grads[o:o + nw].view(L.w.shape), self.grads[o + nw:o + nw + nb]))
            o += nw + nb
        self.m = torch.zeros_like(self.params)
        self.v = torch.zeros_like(self.params)
        ws = max(_lib.size("fpvs_wgrad_workspace_size", L.taps, L.spec.in_channels, L.spec.out_channels, cap)
                 for L in net.layers)
        self.wg_ws = torch.empty(ws, dtype=torch.uint8, device=device)
        self.sums = torch.empty((_lib.size("fpvs_loss_sums_size", B, cap) + 7) // 8, dtype=torch.float64,
                                device=device)
        self.loss = torch.zeros(1, dtype=torch.float64, device=device)
        self.counts = torch.zeros(4 * B, dtype=torch.int64, device=device)
        self.conf_ws = torch.empty(_lib.size("fpvs_bits_confusion_workspace_size", B), dtype=torch.uint8,
                                   device=device)

    # -- forward + loss + backward ------------------------------------------
    def forward_backward(self, bits, gt_bits, stream=None):
        """Loss (device f64, batch mean), hard counts and the flat local-mean gradient."""
        net, lv, tc = self.net, self.lv, self.tcfg
        d = net.cfg.d
        nx, ny, nz = self.grid_dims
        s = _lib.stream_ptr(stream)
        self.maps.run(bits, feat=self.x0, clear=self.pred_bits, stream=stream)
        build_layer_tables(lv, net.kernels(), stream)
        x = self.x0
        for li, (layer, y) in enumerate(zip(net.layers[:-1], self.acts)):
            table, K, masks = layer_table(lv, layer.spec.kernel)
            sp_ = layer.spec
            halo = None
            if self.halo_fwd and self.halo_conv_ws is not None and K == 27 and halo_ok(27, sp_.in_channels,
                                                                                        sp_.out_channels):
                halo = (0, 1, self.halo_conv_ws)
            run_conv(layer, x, x.shape[1], table, K, lv.n, lv.cap, y, y.shape[1], 0, net.precision, stream=stream,
                     masks=masks, halo=halo, halo_tabs=lv.extra.get("halo") if halo else None, settled=li > 0)
            x = y
        run_head(net.layers[-1], x, x.shape[1], lv, d, self.grid_dims, tc.tau, self.pred_bits, self.probs, None,
                 net.precision, stream)
        d3 = self.probs.shape[1]
        _lib.call("fpvs_loss_counts", _lib.ptr(self.probs), d3, _lib.ptr(lv.coords), _lib.ptr(lv.n), lv.cap,
                  _lib.ptr(gt_bits), d, self.B, nx, ny, nz, _lib.ptr(self.sums), s)
        _lib.call("fpvs_loss_grad", _lib.ptr(self.probs), d3, _lib.ptr(lv.coords), _lib.ptr(lv.n), lv.cap,
                  _lib.ptr(gt_bits), d, self.B, nx, ny, nz, _lib.ptr(self.sums), float(tc.alpha), float(tc.lam),
                  _lib.ptr(self.dlogits), _lib.ptr(self.loss), s)
        _lib.call("fpvs_bits_confusion", _lib.ptr(self.pred_bits), _lib.ptr(gt_bits), self.B, self.grid_bytes,
                  _lib.ptr(self.counts), _lib.ptr(self.conf_ws), self.conf_ws.numel(), s)
        self.backward(stream)

    @staticmethod
    def _halo_wgrad_ok(L) -> bool:
        s = L.spec
        return s.kernel == 3 and s.in_channels == 32 and s.out_channels % 8 == 0 and s.out_channels <= 32

    def _tc_backward_ok(self) -> bool:
        # tcgen05 dgrad / wgrad cover 1^3 and 3^3 layers and the fused 1^3 head;
        # other kernel sizes (and a k^3 head) keep the SIMT backward
        layers = self.net.layers
        return (all(L.spec.in_channels % 8 == 0 and L.spec.out_channels % 8 == 0 and L.spec.out_channels <= 256
                    and L.spec.kernel in (1, 3) for L in layers)
                and layers[-1].spec.kernel == 1
                and all(L.spec.in_channels % 32 == 0 for L in layers[1:]))

    def backward(self, stream=None):
        if self.tc_backward:
            return self.backward_tc(stream)
        net, lv = self.net, self.lv
        s = _lib.stream_ptr(stream)
        ins = [self.x0] + self.acts
        dz, lddz = self.dlogits, self.dlogits.shape[1]
        for li in reversed(range(len(net.layers))):
            layer = net.layers[li]
            spec = layer.spec
            x = ins[li]
            table, K, _ = layer_table(lv, spec.kernel)
            dw, db = self.views[li]
            xdt = _lib.F32 if x.dtype == self.dx[0].dtype else _lib.BF16
            _lib.call("fpvs_spconv_wgrad_simt", _lib.ptr(x), x.shape[1], xdt, _lib.ptr(dz), lddz, _lib.ptr(table), K,
                      _lib.ptr(lv.n), lv.cap, spec.in_channels, spec.out_channels, _lib.ptr(dw), _lib.ptr(db),
                      _lib.ptr(self.wg_ws), self.wg_ws.numel(), s)
            if li == 0:
                break
            dx = self.dx[li % 2]
            # relu' of the layer below (z > 0, neural.py:227-228) from its kept output
            _lib.call("fpvs_spconv_dgrad_simt", _lib.ptr(dz), lddz, _lib.ptr(table), K, _lib.ptr(lv.n), lv.cap,
                      _lib.ptr(layer.w), spec.in_channels, spec.out_channels, _lib.ptr(x), xdt, x.shape[1],
                      _lib.ptr(dx), dx.shape[1], s)
            dz, lddz = dx, dx.shape[1]

    def backward_tc(self, stream=None):
        """Tensor-core backward: per layer tcgen05 wgrad (dW, db) and, below the
        first layer, tcgen05 dgrad with the relu' mask fused (bf16 gradients)."""
        net, lv = self.net, self.lv
        s = _lib.stream_ptr(stream)
        ins = [self.x0] + self.acts
        cap = lv.cap
        halo = None
        if self.halo_wgrad:
            halo = sp._halo_tables(lv)  # built by the map build (K3) of this step
        _lib.call("fpvs_cast_bf16_rows", _lib.ptr(self.dlogits), self.dlogits.shape[1], _lib.ptr(lv.n), cap,
                  _lib.ptr(self.dlog16), s)
        dz, lddz = self.dlog16, self.dlog16.shape[1]
        for li in reversed(range(len(net.layers))):
            layer = net.layers[li]
            spec = layer.spec
            x = ins[li]
            table, K = (lv.nbr, 27) if spec.kernel == 3 else (None, 1)
            dw, db = self.views[li]
            if halo is not None and self._halo_wgrad_ok(layer):
                _lib.call("fpvs_spconv_wgrad_halo", _lib.ptr(x), x.shape[1], _lib.ptr(dz), lddz, _lib.ptr(table),
                          _lib.ptr(lv.n), cap, _lib.ptr(halo["rows"]), _lib.ptr(halo["n"]), _lib.ptr(halo["lnbr"]),
                          spec.in_channels, spec.out_channels, _lib.ptr(dw), _lib.ptr(db), _lib.ptr(self.wg_halo_ws),
                          self.wg_halo_ws.numel(), s)
            else:
                _lib.call("fpvs_spconv_wgrad_tc", _lib.ptr(x), x.shape[1], _lib.ptr(dz), lddz, _lib.ptr(table), K,
                          _lib.ptr(lv.n), cap, spec.in_channels, spec.out_channels, _lib.ptr(dw), _lib.ptr(db),
                          _lib.ptr(self.wg_tc_ws), self.wg_tc_ws.numel(), s)
            if li == 0:
                break
            dx = self.dz16[li % 2]
            # dz of the layer below = (dz W'ᵀ on the mirrored map) * relu'(its kept output)
            _lib.call("fpvs_spconv_tc_dgrad", _lib.ptr(dz), lddz, cap, _lib.ptr(table), K,
                      _lib.ptr(lv.nbr_masks if table is not None else None), _lib.ptr(lv.n), cap,
                      _lib.ptr(packed_dgrad_cache(layer, 0, stream)), 0, spec.in_channels, spec.out_channels,
                      _lib.ptr(x), x.shape[1], _lib.ptr(dx), dx.shape[1], s)
            dz, lddz = dx, dx.shape[1]

    # -- exchange + update ---------------------------------------------------
    def pack(self, weight: float = 1.0, samples: int | None = None, stream=None):
        """Scale the local mean gradient by ``weight`` (= B_local / B_global) and
        write the loss / hard-count tail of the exchange buffer.  ``samples`` = 0
        packs an empty share (a rank with no samples in this batch)."""
        B = self.B if samples is None else samples
        if B == 0:
            self.grads.zero_()
        _lib.call("fpvs_exchange_pack", _lib.ptr(self.grads), self.nparams, float(weight), _lib.ptr(self.loss),
                  _lib.ptr(self.counts), B, _lib.stream_ptr(stream))

    def exchange(self, weight: float = 1.0, samples: int | None = None, stream=None):
        """pack() and sum the buffer across ranks: ONE all-reduce per step (NCCL
        over NVLink under torchrun; identity at world size 1)."""
        self.pack(weight, samples, stream)
        dist = _dist()
        if dist is not None and dist.get_world_size() > 1:
            dist.all_reduce(self.grads, op=dist.ReduceOp.SUM)

    def accumulate(self, acc, batch_index: int, stream=None):
        """Add the exchanged tail into the epoch accumulator (device f64[8])."""
        _lib.call("fpvs_exchange_accumulate", _lib.ptr(self.tail), _lib.ptr(acc), int(batch_index),
                  _lib.stream_ptr(stream))

    def update(self, lr: float, step: int, stream=None):
        tc = self.tcfg
        s = _lib.stream_ptr(stream)
        n = self.nparams
        if tc.optimizer == "adamw":
            _lib.call("fpvs_adamw_step", _lib.ptr(self.params), _lib.ptr(self.grads), _lib.ptr(self.m),
                      _lib.ptr(self.v), n, float(lr), 0.9, 0.999, 1e-8, float(tc.weight_decay), int(step), s)
        else:
            _lib.call("fpvs_sgd_step", _lib.ptr(self.params), _lib.ptr(self.grads), n, float(lr), s)
        # every cached bf16 weight image re-packed from the new master weights, one launch
        repack_all(self.net.layers, stream)

    def adopt(self, other: "TrainStep"):
        """Share another plan's flat parameters / optimizer state (a different batch size)."""
        self.params, self.m, self.v = other.params, other.m, other.v
        o = 0
        for L, (dw, db) in zip(self.net.layers, self.views):
            nw, nb = dw.numel(), db.numel()
            L.w = self.params[o:o + nw].view(dw.shape)
            L.b = self.params[o + nw:o + nw + nb]
            L.invalidate()
            o += nw + nb


class Trainer:
    """Holds one TrainStep per local batch size, sharing one parameter set."""

    def __init__(self, net: PvsNet, grid_dims, tcfg: TrainConfig):
        self.net, self.grid_dims, self.tcfg = net, tuple(grid_dims), tcfg
        self.plans = {}
        self.first = None

    def plan(self, B: int) -> TrainStep:
        if B not in self.plans:
            p = TrainStep(self.net, B, self.grid_dims, self.tcfg)
            if self.first is None:
                self.first = p
            else:
                p.adopt(self.first)
            self.plans[B] = p
        return self.plans[B]


def _stack_bits(grids):
    torch = _torch()
    return torch.from_numpy(np.concatenate([g.bits for g in grids])).cuda()


def read_manifest(path):
    """(frame, viewcell, geometry path, gt path) records of a dataset manifest (scenegen.py:433-446)."""
    path = Path(path)
    out = []
    for line in path.read_text().splitlines():
        parts = line.split()
        if not parts or parts[0].startswith("#"):
            continue
        if len(parts) != 4:
            raise ValueError(f"bad manifest record: {line!r}")
        out.append((int(parts[0]), int(parts[1]), str(path.parent / parts[2]), str(path.parent / parts[3])))
    return out


def load_pairs(manifest_path) -> list:
    """(geometry, gt) FroxelGrid pairs of a manifest (neural.py:405-411)."""
    return [(FroxelGrid.load(g), FroxelGrid.load(t)) for _, _, g, t in read_manifest(manifest_path)]


def _rates(tp, fp, fn, gtp):
    if gtp == 0:
        return 0.0, 0.0
    return fn / gtp, fp / gtp


def evaluate_grid_pairs(net: PvsNet, pairs, tau: float, batch: int = 8):
    """Hard FNR/FPR of thresholded predictions over (geometry, gt) FroxelGrid
    pairs (the rates of neural.py:423-439), predicted and counted on packed bits."""
    torch = _torch()
    if not pairs:
        return 0.0, 0.0
    dims = pairs[0][0].dims
    tot = np.zeros(4, dtype=np.int64)
    for i in range(0, len(pairs), batch):
        chunk = pairs[i:i + batch]
        bits = _stack_bits([g for g, _ in chunk])
        gt = _stack_bits([t for _, t in chunk])
        pred = net.predict_bits(bits, len(chunk), dims, tau)
        ws = torch.empty(_lib.size("fpvs_bits_confusion_workspace_size", len(chunk)), dtype=torch.uint8,
                         device="cuda")
        counts = torch.zeros(4 * len(chunk), dtype=torch.int64, device="cuda")
        _lib.call("fpvs_bits_confusion", _lib.ptr(pred), _lib.ptr(gt), len(chunk), bits.numel() // len(chunk),
                  _lib.ptr(counts), _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
        tot += counts.view(-1, 4).sum(0).cpu().numpy()
    return _rates(*[int(v) for v in tot])


def train(pairs, mcfg: ModelConfig, tcfg: TrainConfig, eval_pairs=None, target_fnr: float | None = None,
          target_fpr: float | None = None, checkpoint_path=None, log_path=None, verbose: bool = False,
          precision: str = "fp32"):
    """Mini-batch training over (geometry, gt) FroxelGrid pairs (neural.py:442-510).

    Returns ``(net, history)``.  Under torch.distributed (world > 1) every rank
    calls ``train`` with the same pairs and config; each takes a strided share
    of every global batch and the gradients are all-reduced, so all ranks hold
    identical weights.
    """
    torch = _torch()
    if isinstance(pairs, (str, Path)):
        pairs = load_pairs(pairs)
    if not pairs:
        raise ValueError("no training pairs")
    dims = pairs[0][0].dims
    for g, t in pairs:
        if g.dims != dims or t.dims != dims:
            raise ValueError("all training grids must share one shape")
    dist = _dist()
    rank, world = (dist.get_rank(), dist.get_world_size()) if dist is not None else (0, 1)
    rng = np.random.Generator(np.random.PCG64(tcfg.seed))
    net = PvsNet(mcfg, rng, precision=precision)
    geo = _stack_bits([g for g, _ in pairs])
    lab = _stack_bits([t for _, t in pairs])
    gb = geo.numel() // len(pairs)
    trainer = Trainer(net, dims, tcfg)
    n = len(pairs)
    history, step = [], 0
    # epoch accumulator on the device: loss x samples, samples, TP/FP/FN/GTP,
    # first non-finite batch (-1) and its loss (fpvs_exchange_accumulate)
    acc = torch.zeros(8, dtype=torch.float64, device="cuda")
    for epoch in range(tcfg.epochs):
        order = rng.permutation(n)
        acc.zero_()
        acc[6] = -1.0
        # a step is: forward + loss + backward, pack, ONE all-reduce of the
        # [gradient | loss, counts] buffer, accumulate, optimizer — no host sync
        for start in range(0, n, tcfg.batch_size):
            batch = order[start:start + tcfg.batch_size]
            mine = shard(batch, rank, world)
            if mine:
                plan = trainer.plan(len(mine))
                idx = torch.as_tensor(np.asarray(mine, dtype=np.int64), device="cuda")
                bits = geo.view(n, gb)[idx].reshape(-1)
                gt = lab.view(n, gb)[idx].reshape(-1)
                plan.forward_backward(bits, gt)
                plan.exchange(len(mine) / len(batch))
            else:
                plan = trainer.plan(1)
                plan.exchange(0.0, samples=0)
            plan.accumulate(acc, start // tcfg.batch_size)
            lr = tcfg.lr * (1.0 - tcfg.decay) ** step
            step += 1
            plan.update(lr, step)
        # one host read per epoch; a non-finite loss raises as the reference's
        # per-batch check does (neural.py:478-479), with the same batch index and value
        a = acc.cpu().numpy()
        if a[6] >= 0:
            raise TrainingDiverged(int(a[6]), float(a[7]))
        tot = np.rint(a[2:6]).astype(np.int64)
        fnr, fpr = _rates(*[int(v) for v in tot])
        entry = {"epoch": epoch, "loss": float(a[0]) / max(n, 1), "fnr": fnr, "fpr": fpr}
        if eval_pairs:
            entry["val_fnr"], entry["val_fpr"] = evaluate_grid_pairs(net, eval_pairs, tcfg.tau)
        history.append(entry)
        if verbose and rank == 0:
            print("  ".join(f"{k}={v:.5g}" if isinstance(v, float) else f"{k}={v}" for k, v in entry.items()))
        if (eval_pairs and target_fnr is not None and target_fpr is not None
                and entry["val_fnr"] <= target_fnr and entry["val_fpr"] <= target_fpr):
            break
    if checkpoint_path is not None and rank == 0:
        net.save(checkpoint_path)
    if log_path is not None and rank == 0:
        cols = list(history[0].keys()) if history else ["epoch", "loss", "fnr", "fpr"]
        lines = [",".join(cols)]
        for entry in history:
            lines.append(",".join(f"{entry[c]:.9g}" if isinstance(entry[c], float) else str(entry[c]) for c in cols))
        Path(log_path).write_text("\n".join(lines) + "\n")
    return net, history
