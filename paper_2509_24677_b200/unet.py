"""Config-2 network: 3-level sparse U-Net over 256^3 froxel grids (row UNET).

Not in the reference (its estimator is a dense 3-layer chain,
pkg/src/froxelpvs/neural.py:95-99); BASELINE.json config 2 asks for it and
SURVEY.md §8(a) row UNET pins the architecture, restated in the oracle
(oracle/sparse.py ``unet_forward``):

    L0 (d^3 = 64 ch): subm 64->64, subm 64->64                 = E0
    down k2s2 64->128 -> L1: subm 128->128 x2                  = E1
    down k2s2 128->256 -> L2: subm 256->256 x2
    up k2s2^T 256->128 onto L1 = U1; [E1, U1] -> subm 256->128, 128->128
    up k2s2^T 128->64 onto L0 = U0;  [E0, U0] -> subm 128->64, 64->64
    head 1^3 64->64 + sigmoid + [p >= tau] + deinterleave bit-pack

ReLU after every conv except the head.  Skip concatenation costs nothing:
the encoder output and the up-conv output are written by their producing
kernels into the two column halves of one [rows, 2C] buffer.

A ``UNetPlan`` owns every device buffer for a (B, grid) shape, sized by the
cell-count capacities, so ``run`` is pure kernel launches — no host sync, no
allocation — and can be captured into a CUDA graph.
"""

from __future__ import annotations

import os

import numpy as np

from . import _lib
from . import sparse as sp
from .neural import brick_ok, halo_ok, packed_cache, packed_upblocks_cache, pick_bn, run_conv, run_head


def _torch():
    import torch
    return torch


def layer_table(widths=(64, 128, 256), d3: int = 64):
    c0, c1, c2 = widths
    return (("enc0a", "subm", d3, c0), ("enc0b", "subm", c0, c0), ("down01", "down", c0, c1),
            ("enc1a", "subm", c1, c1), ("enc1b", "subm", c1, c1), ("down12", "down", c1, c2),
            ("enc2a", "subm", c2, c2), ("enc2b", "subm", c2, c2), ("up21", "up", c2, c1),
            ("dec1a", "subm", 2 * c1, c1), ("dec1b", "subm", c1, c1), ("up10", "up", c1, c0),
            ("dec0a", "subm", 2 * c0, c0), ("dec0b", "subm", c0, c0), ("head", "head", c0, d3))


TAPS = {"subm": 27, "down": 8, "up": 8, "head": 1}


class _Spec:
    def __init__(self, cin, cout, act, kernel):
        self.in_channels, self.out_channels, self.activation, self.kernel = cin, cout, act, kernel


class SparseLayer:
    """Weights of one U-Net conv: w (taps*Cin, Cout) f32, row j*Cin + ci."""

    def __init__(self, name, kind, cin, cout, w, b, device="cuda"):
        torch = _torch()
        self.name, self.kind, self.taps = name, kind, TAPS[kind]
        self.spec = _Spec(cin, cout, "sigmoid" if kind == "head" else "relu",
                          {"subm": 3, "down": 2, "up": 2, "head": 1}[kind])
        self.w = torch.as_tensor(np.asarray(w, np.float32)).to(device).contiguous()
        self.b = torch.as_tensor(np.asarray(b, np.float32)).to(device).contiguous()
        self._packed = None

    def packed(self, bn: int = 0, stream=None):
        return packed_cache(self, bn, stream)


class PvsUNet:
    """Sparse U-Net (BASELINE config 2) with Kaiming-uniform init from ``seed``."""

    def __init__(self, seed: int = 1, widths=(64, 128, 256), d: int = 4, precision: str = "bf16",
                 device: str = "cuda", params=None):
        _lib.require_cuda()
        if precision not in ("bf16", "fp32"):
            raise ValueError(f"unknown precision {precision!r}")
        self.d, self.widths, self.precision = d, tuple(widths), precision
        table = layer_table(widths, d ** 3)
        if params is None:
            params = init_params(seed, widths, d ** 3)
        self.layers = {name: SparseLayer(name, kind, cin, cout, *params[name], device=device)
                       for name, kind, cin, cout in table}

    def plan(self, B: int, grid_dims, device="cuda") -> "UNetPlan":
        return UNetPlan(self, B, grid_dims, device)

    def predict_bits(self, bits, B: int, grid_dims, tau: float = 0.5, plan=None, probs=None, logits=None):
        plan = plan or self.plan(B, grid_dims, bits.device)
        out = _torch().empty(B * int(np.prod(grid_dims)) // 8, dtype=_torch().uint8, device=bits.device)
        plan.run(bits, out, tau, probs=probs, logits=logits)
        return out, plan


def init_params(seed: int, widths=(64, 128, 256), d3: int = 64):
    """Kaiming-uniform U(+-sqrt(3 gain / fan_in)) per layer, Generator(PCG64(seed)), layer order."""
    rng = np.random.Generator(np.random.PCG64(seed))
    out = {}
    for name, kind, cin, cout in layer_table(widths, d3):
        fan_in = TAPS[kind] * cin
        gain = 1.0 if kind == "head" else 2.0
        bound = np.sqrt(3.0 * gain / fan_in)
        out[name] = (rng.uniform(-bound, bound, size=(fan_in, cout)), np.zeros(cout))
    return out


class UNetPlan:
    """All device buffers of one (B, grid) frame shape; ``run`` only launches kernels."""

    def __init__(self, net: PvsUNet, B: int, grid_dims, device="cuda"):
        torch = _torch()
        self.net, self.B, self.grid_dims = net, B, tuple(grid_dims)
        d = net.d
        nx, ny, nz = grid_dims
        if nx % 8 or nx % (4 * d) or ny % (4 * d) or nz % (4 * d):
            raise ValueError(f"grid dims {tuple(grid_dims)} must be divisible by 4*d = {4 * d} (and N_x by 8)")
        c0, c1, c2 = net.widths
        self.L0 = sp.new_level(B, (nx // d, ny // d, nz // d), device=device)
        self.L1, self.down01, self.up10 = sp.new_coarse(self.L0)
        self.L2, self.down12, self.up21 = sp.new_coarse(self.L1)
        dt = torch.bfloat16 if net.precision == "bf16" else torch.float32
        e = lambda rows, cols: torch.empty((rows, cols), dtype=dt, device=device)  # noqa: E731
        k0, k1, k2 = self.L0.cap, self.L1.cap, self.L2.cap
        self.x0 = e(k0, d ** 3)
        self.t0a, self.t0b, self.buf0 = e(k0, c0), e(k0, c0), e(k0, 2 * c0)
        self.t1a, self.t1b, self.buf1 = e(k1, c1), e(k1, c1), e(k1, 2 * c1)
        self.t2a, self.t2b = e(k2, c2), e(k2, c2)
        self.bn = {}  # per-layer output-tile width (0 = auto from Cout); see tune()
        # 27-tap layers with 64-multiple channels run the halo-cached kernel
        # (fpvs_spconv_halo); FPVS_HALO=0 keeps them on the plain gather-GEMM
        self.use_halo = net.precision == "bf16" and os.environ.get("FPVS_HALO", "1") != "0"
        # the up convs as one dense GEMM over the coarse rows with a column-block
        # scatter through the down table (fpvs_spconv_tc_upblocks: no sort, no
        # gather); FPVS_UPBLOCKS=0 keeps the parity-sorted gather-GEMM
        self.use_upblocks = net.precision == "bf16" and os.environ.get("FPVS_UPBLOCKS", "1") != "0"
        self.use_upsort = (net.precision == "bf16" and not self.use_upblocks
                           and os.environ.get("FPVS_UPSORT", "1") != "0")
        # the halo tables come out of the fused map build's K3 for the levels in
        # FPVS_MAPS_HALO (default all three: 4 us per frame better than building
        # levels 1 and 2 on the side stream, tools/frame_variant.py)
        self.maps_halo = tuple(int(c) for c in os.environ.get("FPVS_MAPS_HALO", "012")) if self.use_halo else ()
        self.maps = sp.LevelMaps([self.L0, self.L1, self.L2], [self.down01, self.down12], [self.up10, self.up21],
                                 self.grid_dims, d, halo_levels=self.maps_halo, with_up=not self.use_upblocks) \
            if d in (1, 2, 4, 8) else None
        self.level_of = {"enc0a": self.L0, "enc0b": self.L0, "dec0a": self.L0, "dec0b": self.L0,
                         "enc1a": self.L1, "enc1b": self.L1, "dec1a": self.L1, "dec1b": self.L1,
                         "enc2a": self.L2, "enc2b": self.L2}
        self.halo_cfg = {}
        self.halo_ws = None
        # K splits for levels with under a wave of tiles (FPVS_SPLIT=0: none).
        # Unsplit, the streamed e2e gains 2.6 % (4034 -> 4140 grids/s: no
        # partial-sum traffic, other frames fill the idle SMs) but one frame
        # loses 16 us and the fp32 sums change order, so streamed bits would
        # differ near the threshold from the single-frame path; kept on.
        self.allow_split = os.environ.get("FPVS_SPLIT", "1") != "0"
        self._halo_builder = None
        self._up_sorter = None  # parity-sorted up tables (FPVS_UPBLOCKS=0 path; FPVS_UPSORT=0 disables)
        self.overlap = True  # side-stream map tables (see build_maps); device_stage_times turns it off
        # the 1x1x1 head fused into dec0b (FPVS_FUSE_HEAD=0 keeps the stand-alone head launch)
        self.fuse_head = net.precision == "bf16" and os.environ.get("FPVS_FUSE_HEAD", "1") != "0"
        # FPVS_TABLES_SETTLED for the convs after the first (FPVS_SETTLED=0: every conv waits to decode)
        self.settled = os.environ.get("FPVS_SETTLED", "1") != "0"
        # tile-level dataflow between the two convs of a level (fpvs_spconv_halo_flow;
        # FPVS_FLOW=0: grid-wide waits only): per-tile done flags of each producer
        self.flow = self.use_halo and self.settled and os.environ.get("FPVS_FLOW", "1") != "0"
        # level 0 only: its layers run ~2.5 waves of tiles, so the consumer's first
        # tiles fill the producer's last wave; a level-1 pair runs one wave of
        # 111 tiles and measured no faster (dec1b 3 us slower: spinning CTAs)
        self.flow_pairs = {"enc0b": "enc0a", "dec0b": "dec0a"}
        # the first down conv (a plain gather-GEMM) as a consumer of enc0b
        # (fpvs_spconv_tc_flow): measured 2 us slower per frame (enc0b's
        # per-tile publishing outweighs down01's head start), so opt-in only
        self.flow_tc = {"down01": "enc0b"} if os.environ.get("FPVS_FLOW_TC", "0") == "1" else {}
        # the grid writer as a dataflow consumer of dec0b + head
        # (fpvs_rowbits_to_grid_flow; FPVS_GRID_FLOW=0: after dec0b's grid)
        self.grid_flow = self.flow and os.environ.get("FPVS_GRID_FLOW", "1") != "0"
        self.done = {}
        if self.flow:
            for prod in list(self.flow_pairs.values()) + list(self.flow_tc.values()) + \
                    (["dec0b"] if self.grid_flow else []):
                lv = self.level_of[prod]
                self.done[prod] = torch.zeros((lv.cap + 127) // 128, dtype=torch.int32, device=device)
        # the fused head's per-row 64-bit cell masks (fpvs_rowbits_to_grid writes the grid from them)
        self.row_bits = torch.empty(k0, dtype=torch.int64, device=device) if self.fuse_head else None
        self._side = None
        self._side_pending = False
        # 27-tap layers of well-filled levels run the dense-brick conv
        # (fpvs_spconv_brick: 1 x 16 x 8-cell bricks, tap operands straight
        # from a dense halo brick in shared memory, no gather builders);
        # FPVS_BRICK lists the candidate levels, tune() keeps those whose
        # active fraction is >= FPVS_BRICK_MIN; FPVS_BRICK_CFG = "<bn>x<split>".
        # Off by default: on config 2's level 2 (90 % active) the frame
        # measured 315 us against 309 with the halo kernel
        self.brick_levels = tuple(int(c) for c in os.environ.get("FPVS_BRICK", "")) if self.use_halo else ()
        self.brick_min = float(os.environ.get("FPVS_BRICK_MIN", "0.5"))
        self.brick_cfg = tuple(int(v) for v in os.environ.get("FPVS_BRICK_CFG", "128x2").split("x"))
        self.brick_of = {}
        self.brick_ws = {}
        if self.use_halo:
            self.set_halo({k: lv.cap for k, lv in self.level_of.items()})

    def set_halo(self, rows: dict, cfg: dict | None = None):
        """(bn, split) per halo layer: bn = 128 when Cout allows, split so the
        layer has about two waves of work units; ``cfg`` overrides."""
        torch = _torch()
        self.halo_cfg = {}
        need = {}  # one workspace per level: layers of a level share (cap, Cout, bn, split)
        for name, r in rows.items():
            layer = self.net.layers[name]
            cin, cout = layer.spec.in_channels, layer.spec.out_channels
            if not halo_ok(27, cin, cout):
                continue
            # measured on config 2 in the whole flushed frame (tools/split_frame.py):
            # 128-wide tiles; a 2-way K split only where the level has well under
            # a wave of tiles (level 2); every other split, including the
            # last-wave tail split (-2) of dec0a, costs 4-80 us per frame
            bn = 128 if cout % 128 == 0 else 64
            tiles = max(1, (r + 127) // 128) * (cout // bn)
            split = 2 if (tiles * 2 <= 148 and self.allow_split) else 1
            if cfg and name in cfg:
                bn, split = cfg[name]
            self.halo_cfg[name] = (bn, split)
            lv = self.level_of[name]
            key = id(lv)
            need[key] = max(need.get(key, 256),
                            _lib.size("fpvs_spconv_halo_workspace_size", lv.cap, cout, bn, split))
        if self.halo_ws is None:
            self.halo_ws = {}
        for key, nbytes in need.items():
            if key not in self.halo_ws or self.halo_ws[key].numel() < nbytes:
                self.halo_ws[key] = torch.zeros(nbytes, dtype=torch.uint8, device=self.L0.coords.device)
            else:
                self.halo_ws[key].zero_()  # the counter region moves with the split mode

    def tune(self, bits):
        """Pick per-layer tile widths from one frame's active counts (one host sync).

        Layers whose rows make fewer than one wave of 128-row tiles split N
        across CTAs; reuse the plan for frames of similar occupancy.
        """
        self.build_maps(bits)
        n0, n1, n2 = self.counts()
        rows = {"enc0a": n0, "enc0b": n0, "down01": n1, "enc1a": n1, "enc1b": n1, "down12": n2, "enc2a": n2,
                "enc2b": n2, "up21": n1, "dec1a": n1, "dec1b": n1, "up10": n0, "dec0a": n0, "dec0b": n0}
        self.bn = {k: pick_bn(self.net.layers[k].spec.out_channels, v) for k, v in rows.items()}
        if self.use_halo:
            self.set_halo({k: rows[k] for k in self.level_of})
            self.set_bricks((n0, n1, n2))
        return self.bn

    def set_bricks(self, counts, cfg: dict | None = None):
        """The dense-brick conv for the 27-tap layers of FPVS_BRICK levels whose
        active fraction is >= brick_min; ``cfg`` maps layer -> (bn, split)."""
        torch = _torch()
        self.brick_of = {}
        for name, lv in self.level_of.items():
            li = int(name[-2])
            if cfg is None and (li not in self.brick_levels or counts[li] < self.brick_min * lv.ncells):
                continue
            if cfg is not None and name not in cfg:
                continue
            spec = self.net.layers[name].spec
            bn, split = cfg[name] if cfg is not None else self.brick_cfg
            if not brick_ok(27, spec.in_channels, spec.out_channels) or spec.out_channels % bn or \
                    (spec.in_channels // 64) % split:
                continue
            X, Y, Z = lv.dims
            nbytes = _lib.size("fpvs_spconv_brick_workspace_size", lv.B, X, Y, Z, spec.out_channels, bn, split)
            ws = self.brick_ws.get(name)
            if ws is None or ws.numel() < max(nbytes, 256):
                ws = self.brick_ws[name] = torch.zeros(max(nbytes, 256), dtype=torch.uint8, device=lv.coords.device)
            self.brick_of[name] = (bn, split)

    def build_maps(self, bits, gather: bool = False, clear=None):
        """Level hierarchy + tables (three fused launches); with ``gather`` also the
        level-0 features, and ``clear`` (the output grid) is zeroed on the way."""
        if self.maps is not None:
            self.maps.run(bits, self.x0 if gather else None, 0, clear)
        else:
            sp.fill_level_from_bits(self.L0, bits, self.grid_dims, self.net.d)
            sp.fill_coarse(self.L0, self.L1, self.down01, self.up10)
            sp.fill_coarse(self.L1, self.L2, self.down12, self.up21)
        if self.use_halo:
            if self._halo_builder is None:
                self._halo_builder = sp.HaloBuilder([self.L0])
                side = [lv for i, lv in ((1, self.L1), (2, self.L2)) if self.maps is None or i not in self.maps_halo]
                self._halo_builder_coarse = sp.HaloBuilder(side) if side else None
            if self.maps is None:
                self._halo_builder.run()  # level 0: needed by the first conv (else built by the fused maps)
        # the up-sort tables and the level-1/2 halo tables are first used by
        # enc1a / up21: with ``overlap`` they run on a side stream, filling SMs
        # the level-0 convs leave idle at their tails (joined before enc1a)
        torch = _torch()
        side = self.overlap and (self.use_upsort or (self.use_halo and self._halo_builder_coarse is not None))
        if side:
            if self._side is None:
                self._side = torch.cuda.Stream()
                self._ev_maps, self._ev_side = torch.cuda.Event(), torch.cuda.Event()
            self._ev_maps.record()
            self._side.wait_event(self._ev_maps)
            ctx = torch.cuda.stream(self._side)
        else:
            import contextlib
            ctx = contextlib.nullcontext()
        with ctx:
            if self.use_upsort:
                if self._up_sorter is None:
                    self._up_sorter = sp.UpSorter([(self.L1, self.up21), (self.L0, self.up10)])
                self._up_sorter.run()
            if self.use_halo and self._halo_builder_coarse is not None:
                self._halo_builder_coarse.run()
        if side:
            self._ev_side.record(self._side)
            self._side_pending = True

    def _join_side(self):
        if self._side_pending:
            _torch().cuda.current_stream().wait_event(self._ev_side)
            self._side_pending = False

    def stages(self, bits, out_bits, tau: float = 0.5, probs=None, logits=None, maps: bool = True):
        """The frame as an ordered list of (stage name, launch function).

        Each function only enqueues kernels and is idempotent, so a stage can be
        replayed on its own (per-stage device timing) or all run in order.
        """
        net, P = self.net, self.net.precision
        L = net.layers
        L0, L1, L2 = self.L0, self.L1, self.L2
        c0, c1, c2 = net.widths
        d3 = net.d ** 3
        out = []
        fused = maps and self.maps is not None
        # the head fused into dec0b's epilogue (fpvs_spconv_halo_head): the
        # activations never leave the SM and each active cell's 64 threshold
        # bits go out as one word, which fpvs_rowbits_to_grid turns into every
        # word of the output grid (no clear); taken for thresholded bits only
        # (probabilities / logits keep the stand-alone head)
        hc0 = self.halo_cfg.get("dec0b")
        nx, ny, nz = self.grid_dims
        fuse_head = (self.fuse_head and fused and hc0 is not None and hc0 == (64, 1) and c0 == 64 and net.d == 4
                     and nx % 32 == 0 and probs is None and logits is None and 0.0 < float(tau) < 1.0)
        if fused:
            # maps + level-0 features (+ clearing the output grid for the
            # stand-alone head's scatter): three launches
            clear = None if fuse_head else out_bits
            out.append(("maps", lambda: self.build_maps(bits, gather=True, clear=clear)))
        else:
            if maps:
                out.append(("maps", lambda: self.build_maps(bits)))
            out.append(("gather", lambda: sp.gather_features(bits, L0, self.grid_dims, net.d, self.x0.dtype,
                                                             out=self.x0)))

        # dataflow pairs usable with this plan's tile settings: the producer
        # runs unsplit full-width tiles, both convs are halo convs, and the
        # consumer's weights are packed now (before the frame's launches)
        flow_in = {}
        if self.flow and fused:
            for cons, prod in self.flow_pairs.items():
                pc, cc = self.halo_cfg.get(prod), self.halo_cfg.get(cons)
                if pc and cc and pc == (L[prod].spec.out_channels, 1):
                    flow_in[cons] = self.done[prod]
                    L[cons].packed(cc[0])
                    if cons == "dec0b":
                        L["head"].packed(64)  # the fused head's weights (read without a grid-wide wait)
        flow_out = {self.flow_pairs[c]: self.done[self.flow_pairs[c]] for c in flow_in}
        flow_tc, flow_n = {}, {}
        if self.flow and fused:
            for cons, prod in self.flow_tc.items():
                pc = self.halo_cfg.get(prod)
                if pc and pc == (L[prod].spec.out_channels, 1):
                    flow_tc[cons] = self.done[prod]
                    flow_n[cons] = self.level_of[prod].n
                    flow_out[prod] = self.done[prod]
                    L[cons].packed(self.bn.get(cons, 0))

        def conv(name, x, ldx, table, K, lv, y, ldy, off=0, masks=None):
            def launch():
                if name == "enc1a":
                    self._join_side()
                hc = self.halo_cfg.get(name) if K == 27 else None
                halo = (hc[0], hc[1], self.halo_ws[id(lv)]) if hc else None
                if self.use_upblocks and name in ("up21", "up10"):
                    coarse, child = (L2, self.down12) if name == "up21" else (L1, self.down01)
                    layer = L[name]
                    # 256-wide tiles (measured faster than 128 / 64, tools/frame_variant.py)
                    w8, b8 = packed_upblocks_cache(layer, 256)
                    _lib.call("fpvs_spconv_tc_upblocks", _lib.ptr(x), ldx, x.shape[0], _lib.ptr(coarse.n), coarse.cap,
                              _lib.ptr(w8), 256, _lib.ptr(b8), layer.spec.in_channels, layer.spec.out_channels,
                              _lib.ACT["relu"], _lib.ptr(child), _lib.ptr(y), ldy, off, _lib.stream_ptr())
                    return
                us = lv.extra.get("upsort") if (self.use_upsort and name in ("up21", "up10")) else None
                if us is not None:
                    run_conv(L[name], x, ldx, us["table"], K, us["n"], us["cap"], y, ldy, off, P, act="relu",
                             bn=self.bn.get(name, 0), masks=us["masks"], out_rows=us["perm"])
                    return
                bc = self.brick_of.get(name) if K == 27 else None
                if bc is not None:
                    run_conv(L[name], x, ldx, table, K, lv.n, lv.cap, y, ldy, off, P, act="relu",
                             brick=(bc[0], bc[1], self.brick_ws[name], lv), settled=self.settled)
                    return
                # every conv but the first reads tables the map build wrote two or more launches back
                run_conv(L[name], x, ldx, table, K, lv.n, lv.cap, y, ldy, off, P, act="relu", bn=self.bn.get(name, 0),
                         masks=masks, halo=halo, halo_tabs=lv.extra.get("halo") if hc else None,
                         settled=name != "enc0a" and self.settled,
                         done_out=flow_out.get(name) if hc else None,
                         done_in=flow_in.get(name) if hc else flow_tc.get(name), done_n=flow_n.get(name))
            out.append((name, launch))

        m0, m1, m2 = L0.nbr_masks, L1.nbr_masks, L2.nbr_masks
        dm01, um10 = L1.extra["down_masks"], L1.extra["up_masks"]
        dm12, um21 = L2.extra["down_masks"], L2.extra["up_masks"]
        conv("enc0a", self.x0, d3, L0.nbr, 27, L0, self.t0a, c0, masks=m0)
        conv("enc0b", self.t0a, c0, L0.nbr, 27, L0, self.buf0, 2 * c0, 0, m0)          # E0 -> buf0[:, :c0]
        conv("down01", self.buf0, 2 * c0, self.down01, 8, L1, self.t1a, c1, masks=dm01)
        conv("enc1a", self.t1a, c1, L1.nbr, 27, L1, self.t1b, c1, masks=m1)
        conv("enc1b", self.t1b, c1, L1.nbr, 27, L1, self.buf1, 2 * c1, 0, m1)          # E1 -> buf1[:, :c1]
        conv("down12", self.buf1, 2 * c1, self.down12, 8, L2, self.t2a, c2, masks=dm12)
        conv("enc2a", self.t2a, c2, L2.nbr, 27, L2, self.t2b, c2, masks=m2)
        conv("enc2b", self.t2b, c2, L2.nbr, 27, L2, self.t2a, c2, masks=m2)
        conv("up21", self.t2a, c2, self.up21, 8, L1, self.buf1, 2 * c1, c1, um21)       # U1 -> buf1[:, c1:]
        conv("dec1a", self.buf1, 2 * c1, L1.nbr, 27, L1, self.t1a, c1, masks=m1)
        conv("dec1b", self.t1a, c1, L1.nbr, 27, L1, self.t1b, c1, masks=m1)
        conv("up10", self.t1b, c1, self.up10, 8, L0, self.buf0, 2 * c0, c0, um10)       # U0 -> buf0[:, c0:]
        conv("dec0a", self.buf0, 2 * c0, L0.nbr, 27, L0, self.t0a, c0, masks=m0)
        if fuse_head:
            def dec0b_head():
                hl = L["head"]
                ht = L0.extra["halo"]
                ws = self.halo_ws[id(L0)]
                args = [_lib.ptr(self.t0a), c0, self.t0a.shape[0], _lib.ptr(L0.nbr), _lib.ptr(ht["lnbr"]),
                        _lib.ptr(ht["rows"]), _lib.ptr(ht["n"]), _lib.ptr(m0), _lib.ptr(L0.n), L0.cap,
                        _lib.ptr(L["dec0b"].packed(64)), _lib.ptr(L["dec0b"].b), c0, _lib.ptr(ws), ws.numel(),
                        _lib.ptr(hl.packed(64)), _lib.ptr(hl.b), float(tau), _lib.ptr(self.row_bits),
                        _lib.TABLES_SETTLED if self.settled else 0, _lib.ptr(flow_in.get("dec0b"))]
                if grid_done is not None:
                    _lib.call("fpvs_spconv_halo_head_flow", *args, _lib.ptr(grid_done), _lib.stream_ptr())
                else:
                    _lib.call("fpvs_spconv_halo_head", *args, _lib.stream_ptr())

            # the grid writer waits only for the dec0b tiles its cells' rows lie in
            grid_done = self.done.get("dec0b") if (self.grid_flow and self.settled and nz // 4 <= 256) else None

            def grid_writer():
                if grid_done is not None:
                    _lib.call("fpvs_rowbits_to_grid_flow", _lib.ptr(self.row_bits), _lib.ptr(L0.index_vol), self.B,
                              nx, ny, nz, net.d, _lib.ptr(out_bits), _lib.ptr(grid_done), _lib.stream_ptr())
                else:
                    _lib.call("fpvs_rowbits_to_grid", _lib.ptr(self.row_bits), _lib.ptr(L0.index_vol), self.B, nx,
                              ny, nz, net.d, _lib.ptr(out_bits), _lib.stream_ptr())
            out.append(("dec0b", dec0b_head))
            out.append(("grid", grid_writer))  # its own stage: per-stage times keep it out of dec0b's
            return out
        conv("dec0b", self.t0a, c0, L0.nbr, 27, L0, self.t0b, c0, masks=m0)

        def head():
            if not fused:
                out_bits.zero_()
            run_head(L["head"], self.t0b, c0, L0, net.d, self.grid_dims, tau, out_bits, probs, logits, P)
        out.append(("head", head))
        return out

    def run(self, bits, out_bits, tau: float = 0.5, probs=None, logits=None, maps: bool = True, events=None):
        """One frame: maps, sparse interleave, 14 convs, fused head into ``out_bits`` (zeroed here).

        ``events`` (a list) receives (stage, cuda.Event) marks (host-launch timing).
        """
        from .pipeline import _ev
        for name, fn in self.stages(bits, out_bits, tau, probs, logits, maps):
            _ev(events, name)
            fn()
        _ev(events, "end")

    def layer_flops(self):
        """Algorithmic FLOPs per conv of the last frame (2 * pairs * Cin * Cout; no zero-fill)."""
        n0, n1, n2 = self.counts()
        p0 = int((self.L0.nbr[:n0] >= 0).sum())
        p1 = int((self.L1.nbr[:n1] >= 0).sum())
        p2 = int((self.L2.nbr[:n2] >= 0).sum())
        c0, c1, c2 = self.net.widths
        d3 = self.net.d ** 3
        return {"enc0a": 2 * p0 * d3 * c0, "enc0b": 2 * p0 * c0 * c0, "down01": 2 * n0 * c0 * c1,
                "enc1a": 2 * p1 * c1 * c1, "enc1b": 2 * p1 * c1 * c1, "down12": 2 * n1 * c1 * c2,
                "enc2a": 2 * p2 * c2 * c2, "enc2b": 2 * p2 * c2 * c2, "up21": 2 * n1 * c2 * c1,
                "dec1a": 2 * p1 * 2 * c1 * c1, "dec1b": 2 * p1 * c1 * c1, "up10": 2 * n0 * c1 * c0,
                "dec0a": 2 * p0 * 2 * c0 * c0, "dec0b": 2 * p0 * c0 * c0, "head": 2 * n0 * c0 * d3}

    def counts(self):
        return self.L0.count(), self.L1.count(), self.L2.count()

    def useful_flops(self):
        return sum(self.layer_flops().values())
