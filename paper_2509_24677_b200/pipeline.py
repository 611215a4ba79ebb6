"""Frame pipelines: preallocated plans replayed as CUDA graphs.

``predict_pvs`` (pkg/src/froxelpvs/neural.py:513-526) is interleave ->
forward -> deinterleave(tau) per grid.  On the device that is ~35 kernel
launches per frame (maps, sparse interleave, convs, fused head), each a few
microseconds, so the host would dominate if it launched them one by one.  A
``FramePipeline`` allocates every buffer once for a (B, grid) shape, runs the
frame eagerly once (warm-up: lazily packed weights, kernel attributes), then
captures it into one CUDA graph.  ``run_device`` replays the graph on
device-resident packed bits; ``infer`` adds the pinned host <-> device copies
of the packed input and output grids (Nx*Ny*Nz/8 bytes each way).
"""

from __future__ import annotations

import numpy as np

from . import sparse as sp
from .neural import PvsNet, build_layer_tables, layer_table, run_conv, run_head


def _torch():
    import torch
    return torch


class _NoGC:
    """Garbage collection off while a CUDA graph is captured: a collected
    CUDAGraph from earlier work would be destroyed mid-capture, which CUDA
    forbids (cudaErrorStreamCaptureUnsupported)."""

    def __enter__(self):
        import gc
        self._was = gc.isenabled()
        gc.collect()
        gc.disable()

    def __exit__(self, *exc):
        import gc
        if self._was:
            gc.enable()
        return False


no_gc = _NoGC


class ChainPlan:
    """Buffers for a linear PvsNet (configs 1, 3, 4, 5) over B packed grids."""

    def __init__(self, net: PvsNet, B: int, grid_dims, device="cuda", cap: int | None = None):
        torch = _torch()
        self.net, self.B, self.grid_dims = net, B, tuple(grid_dims)
        d = net.cfg.d
        nx, ny, nz = grid_dims
        if nx % 8 or nx % d or ny % d or nz % d:
            raise ValueError(f"grid dims {tuple(grid_dims)} not divisible by interleave factor {d} (N_x by 8)")
        self.L0 = sp.new_level(B, (nx // d, ny // d, nz // d), cap, device=device)
        dt = torch.bfloat16 if net.precision == "bf16" else torch.float32
        widest = max(s.out_channels for s in net.cfg.layers[:-1]) if len(net.cfg.layers) > 1 else 1
        k = self.L0.cap
        self.x0 = torch.empty((k, d ** 3), dtype=dt, device=device)
        self.ping = torch.empty((k, widest), dtype=dt, device=device)
        self.pong = torch.empty((k, widest), dtype=dt, device=device)
        # the fused level build (levels.cu: three launches for flags, compaction,
        # tables + features + output clear) where the grid shape allows it
        try:
            self.maps = sp.LevelMaps([self.L0], [], [], self.grid_dims, d)
        except ValueError:
            self.maps = None

    def stages(self, bits, out_bits, tau: float = 0.5, probs=None, logits=None):
        """Ordered (name, idempotent launch function) list of one frame."""
        net, lv = self.net, self.L0
        d = net.cfg.d
        kernels = net.kernels()

        def tables():
            build_layer_tables(lv, kernels)  # k^3 maps of k not in {1, 3} (none for configs 1-5)
        if self.maps is not None:
            # maps + sparse interleave + clearing the output grid in one fused build
            out = [("maps", lambda: (self.maps.run(bits, self.x0, d ** 3, out_bits), tables()))]
        else:
            out = [("maps", lambda: (sp.fill_level_from_bits(lv, bits, self.grid_dims, d), tables())),
                   ("gather", lambda: sp.gather_features(bits, lv, self.grid_dims, d, self.x0.dtype, out=self.x0))]
        x, ldx = self.x0, d ** 3
        bufs = (self.ping, self.pong)
        for i, layer in enumerate(net.layers[:-1]):
            y = bufs[i % 2]
            table, K, masks = layer_table(lv, layer.spec.kernel)
            out.append((f"conv{i}", lambda layer=layer, x=x, ldx=ldx, table=table, K=K, y=y, masks=masks:
                        run_conv(layer, x, ldx, table, K, lv.n, lv.cap, y, y.shape[1], 0, net.precision,
                                 masks=masks)))
            x, ldx = y, y.shape[1]

        def head(x=x, ldx=ldx):
            if self.maps is None:
                out_bits.zero_()  # else cleared by the fused map build
            run_head(net.layers[-1], x, ldx, lv, d, self.grid_dims, tau, out_bits, probs, logits, net.precision)
        out.append(("head", head))
        return out

    def run(self, bits, out_bits, tau: float = 0.5, probs=None, logits=None, events=None):
        for name, fn in self.stages(bits, out_bits, tau, probs, logits):
            _ev(events, name)
            fn()
        _ev(events, "end")

    def layer_flops(self):
        n = self.L0.count()
        p = int((self.L0.nbr[:n] >= 0).sum())
        return {f"conv{i}": 2 * (p if layer.spec.kernel == 3 else n) * layer.spec.in_channels
                * layer.spec.out_channels for i, layer in enumerate(self.net.layers[:-1])} | {
            "head": 2 * n * self.net.layers[-1].spec.in_channels * self.net.layers[-1].spec.out_channels}

    def counts(self):
        return (self.L0.count(),)

    def useful_flops(self):
        n = self.L0.count()
        p = int((self.L0.nbr[:n] >= 0).sum())
        f = 0
        for layer in self.net.layers:
            s = layer.spec
            f += 2 * (p if s.kernel == 3 else n) * s.in_channels * s.out_channels
        return f


def _ev(events, name):
    """Record a CUDA event named ``name`` on the current stream (stage timing)."""
    if events is None:
        return
    torch = _torch()
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    events.append((name, e))


def stage_times(events):
    """[(stage, ms)] between consecutive recorded events (includes host launch gaps)."""
    return [(a[0], a[1].elapsed_time(b[1])) for a, b in zip(events, events[1:])]


def device_stage_times(plan, bits, out_bits, tau: float = 0.5, reps: int = 20, flush=None):
    """Per-stage DEVICE time (ms): each stage captured alone into a CUDA graph of
    ``reps`` back-to-back copies and replayed, so host launch overhead is
    excluded.  ``flush`` (a buffer > L2) is cleared before each replay."""
    torch = _torch()
    res = {}
    saved = getattr(plan, "overlap", None)
    if saved is not None:
        plan.overlap = False  # each stage is captured alone: no cross-stage side stream
    for name, fn in plan.stages(bits, out_bits, tau):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s), no_gc():
            with torch.cuda.graph(g, stream=s):
                for _ in range(reps):
                    fn()
        torch.cuda.current_stream().wait_stream(s)
        times = []
        for _ in range(3):
            if flush is not None:
                flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) / reps)
        res[name] = min(times)
        del g
    if saved is not None:
        plan.overlap = saved
    return res


def frame_stage_times(plan, bits, out_bits, tau: float = 0.5, flush=None, reps: int = 10):
    """Per-stage DEVICE time (ms) inside the real, L2-flushed frame.

    Prefix differencing: for k = 1..S the first k stages are captured as one
    CUDA graph (exactly the benchmarked frame's launches, PDL overlap and
    side-stream fork/join included, no timing nodes inside) and timed with
    events around each replay after an untimed L2 flush (``flush``, larger
    than the L2); stage k's time is T_k - T_{k-1} (medians over ``reps``), so
    the stages sum to the frame time.  (Timing events BETWEEN stages were
    measured to add ~7 us per boundary — they break PDL overlap — and L2-warm
    isolated replays to undercount it.)  The U-Net's side-stream map tables
    are serialised into "maps" here (``overlap`` off), or their join would be
    charged to whichever conv a prefix happens to end on.  Returns
    (per-stage dict, frame ms of this serialised frame).
    """
    torch = _torch()
    saved = getattr(plan, "overlap", None)
    if saved is not None:
        plan.overlap = False
    try:
        return _prefix_times(plan, bits, out_bits, tau, flush, reps)
    finally:
        if saved is not None:
            plan.overlap = saved


def _prefix_times(plan, bits, out_bits, tau, flush, reps):
    torch = _torch()
    stages = plan.stages(bits, out_bits, tau)
    for _, fn in stages:
        fn()
    join = getattr(plan, "_join_side", None)
    if join is not None:
        join()
    torch.cuda.synchronize()
    prefix = [0.0]
    for k in range(1, len(stages) + 1):
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s), no_gc():
            with torch.cuda.graph(g, stream=s):
                for _, fn in stages[:k]:
                    fn()
                if join is not None:
                    join()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            if flush is not None:
                flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        prefix.append(float(np.median(ts)))
        del g
    per = {name: max(prefix[i + 1] - prefix[i], 0.0) for i, (name, _) in enumerate(stages)}
    return per, prefix[-1]


class FramePipeline:
    """CUDA-graph replay of one frame for a fixed (B, grid) shape.

    ``net`` is a PvsUNet (config 2) or a PvsNet (configs 1/3/4).  The input
    is ``self.in_bits`` (packed grids, device), the output ``self.out_bits``.
    """

    def __init__(self, net, B: int, grid_dims, tau: float = 0.5, graph: bool = True, device="cuda"):
        torch = _torch()
        self.net, self.B, self.grid_dims, self.tau = net, B, tuple(grid_dims), float(tau)
        nbytes = B * int(np.prod(grid_dims)) // 8
        self.plan = net.plan(B, grid_dims, device) if hasattr(net, "plan") else ChainPlan(net, B, grid_dims, device)
        self.in_bits = torch.zeros(nbytes, dtype=torch.uint8, device=device)
        self.out_bits = torch.zeros(nbytes, dtype=torch.uint8, device=device)
        self.graph = None
        self._use_graph = graph

    def load(self, bits):
        self.in_bits.copy_(bits, non_blocking=True)

    def capture(self, tune: bool = True):
        """Tune tile widths on the loaded frame, warm up eagerly, capture a CUDA graph."""
        torch = _torch()
        if tune and hasattr(self.plan, "tune"):
            self.plan.tune(self.in_bits)
        self.plan.run(self.in_bits, self.out_bits, self.tau)
        torch.cuda.synchronize()
        if not self._use_graph:
            return
        self.graph = self._capture(self.in_bits, self.out_bits)

    def _capture(self, in_bits, out_bits):
        torch = _torch()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s), no_gc():
            with torch.cuda.graph(g, stream=s):
                self.plan.run(in_bits, out_bits, self.tau)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        return g

    def run_device(self):
        if self.graph is not None:
            self.graph.replay()
        else:
            self.plan.run(self.in_bits, self.out_bits, self.tau)
        return self.out_bits

    def infer(self, host_bits, host_out=None):
        """Host packed grids in, host packed PVS out (pinned buffers avoid staging)."""
        torch = _torch()
        src = torch.as_tensor(host_bits)
        self.in_bits.copy_(src, non_blocking=True)
        self.run_device()
        if host_out is None:
            host_out = torch.empty(self.out_bits.numel(), dtype=torch.uint8, pin_memory=True)
        host_out.copy_(self.out_bits, non_blocking=True)
        return host_out

    # -- streaming: frames in flight on separate compute streams ------------
    # Lane k (k < inflight) is a FramePipeline with its own buffers, CUDA graph
    # and compute stream; frame i runs on lane i % inflight.  With several
    # frames in flight the lanes run WITHOUT the level-0 tile dataflow: its
    # early-resident consumer CTAs wait on SMs another frame would use
    # (measured 3980 -> 4035 grids/s at 4 in flight); one frame in flight keeps
    # this pipeline (dataflow on, the lower latency).
    # Uploads and downloads go through two shared copy streams, so frame i's
    # compute overlaps frame i+1's upload, frame i-1's download and, with
    # inflight >= 2, the other lanes' compute: the level-1/2 convs leave SMs
    # idle (111 and 29 row tiles for 148 SMs) that the next frame fills.
    def _ensure_streaming(self, inflight: int):
        lanes = getattr(self, "_lanes", None)
        if lanes is not None and len(lanes) == inflight:
            return
        torch = _torch()
        if self.graph is None:
            self.capture(tune=False)
        if inflight == 1 or not getattr(self.plan, "flow", False):
            pipes = [self]
        else:
            pipes = []
        while len(pipes) < inflight:
            p = FramePipeline(self.net, self.B, self.grid_dims, self.tau, graph=self._use_graph)
            if inflight > 1:
                # concurrent frames fill each other's idle SMs: no spinning
                # dataflow consumers (conv pairs, grid writer) in the lanes
                p.plan.flow = False
                p.plan.grid_flow = False
            p.in_bits.copy_(self.in_bits)
            p.capture()
            pipes.append(p)
        self._lanes = [{"pipe": p, "comp": torch.cuda.Stream(), "h2d": torch.cuda.Event(),
                        "done": torch.cuda.Event(), "d2h": torch.cuda.Event()} for p in pipes]
        self._h2d, self._d2h = torch.cuda.Stream(), torch.cuda.Stream()

    def infer_stream(self, host_ins, host_outs, inflight: int = 2):
        """Frames ``host_ins[i]`` (pinned packed grids) -> ``host_outs[i]`` (pinned).

        Every frame is uploaded, run and downloaded; up to ``inflight`` frames
        compute concurrently (separate buffers), copies overlap compute.
        Enqueues relative to the current stream (which joins every stream used
        at the end); the caller synchronises."""
        torch = _torch()
        self._ensure_streaming(max(1, int(inflight)))
        cur = torch.cuda.current_stream()
        lanes = self._lanes
        for ln in lanes:
            ln["done"].record(cur)
            ln["d2h"].record(cur)
        self._h2d.wait_stream(cur)
        self._d2h.wait_stream(cur)
        for i, (hin, hout) in enumerate(zip(host_ins, host_outs)):
            ln = lanes[i % len(lanes)]
            p, comp = ln["pipe"], ln["comp"]
            self._h2d.wait_event(ln["done"])  # the lane's previous frame no longer reads in_bits
            with torch.cuda.stream(self._h2d):
                p.in_bits.copy_(torch.as_tensor(hin), non_blocking=True)
            ln["h2d"].record(self._h2d)
            comp.wait_event(ln["h2d"])
            comp.wait_event(ln["d2h"])  # the lane's previous result has left out_bits
            with torch.cuda.stream(comp):
                if p.graph is not None:
                    p.graph.replay()
                else:
                    p.plan.run(p.in_bits, p.out_bits, p.tau)
            ln["done"].record(comp)
            self._d2h.wait_event(ln["done"])
            with torch.cuda.stream(self._d2h):
                hout.copy_(p.out_bits, non_blocking=True)
            ln["d2h"].record(self._d2h)
        for ln in lanes:
            cur.wait_stream(ln["comp"])
        cur.wait_stream(self._d2h)
        cur.wait_stream(self._h2d)
        return host_outs
