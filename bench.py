"""NeuralPVS hot-path benchmark (BASELINE.json metric: froxel grids/s and
ms/frame at 256^3, bs1, per GPU count; % of tensor-pipe peak).

Workload (BASELINE config 2): one 256^3 froxel grid per step per GPU (4000
seeded boxes, edges 1-12, seed 1), interleave d=4 -> 64^3 cells x 64 ch,
3-level sparse U-Net (64/128/256 ch), bf16 activations/weights with fp32
accumulation, fused sigmoid + threshold + deinterleave bit-pack.  A step is
one whole frame: kernel maps (3 levels + parity-sorted up tables + per-tile
halo tables), sparse interleave, 14 convs, head.

* ``value``: frames with the packed input already in HBM, each step replayed
  from one CUDA graph; L2 is flushed (256 MiB memset, untimed) before every
  step; device time from CUDA events on the launching stream, max over ranks.
* ``e2e``: the same frames through ``FramePipeline.infer_stream`` — pinned
  host packed grid -> H2D -> frame -> D2H packed PVS for every step, every
  copy inside the timed region; up to E2E_INFLIGHT = 4 frames compute
  concurrently on separate streams with separate buffers (each frame is
  still one bs1 pass).  ``e2e.latency_ms``: one frame in flight, pinned host
  in -> device -> packed PVS back on the host, synchronised per frame (the
  bs1 ms/frame of the metric, end to end).
* ``roofline``: the dominant kernel, the tcgen05 sparse conv (14 launches per
  frame: 10 halo-cached subm convs and 4 down/up gather-GEMMs): algorithmic
  FLOPs (2 * present pairs * Cin * Cout; zero-filled taps not counted) / its
  per-launch device time measured INSIDE the L2-flushed frame
  (``pipeline.frame_stage_times``: the frame as one CUDA graph with timing
  events between stages).  ``traffic`` = DRAM bytes per conv launch from the
  committed ncu --set full capture (profiles/).
* ``cpu_baseline``: the numpy sparse restatement (oracle/, fp64) of the same
  frame on this host's cores (rank 0, N=1).
* ``config3`` (side line, every N): BASELINE config 3, 64 independent config-1
  grids sharded over the ranks — rank r runs grids [r*64/N, (r+1)*64/N) as
  one batched frame (CUDA graph, L2 flushed between steps), no collective on
  the data path; grids/s = 64 * steps / max-rank time.
* ``train_config5`` (side line, every N): BASELINE config 5, 8 x 128^3 grids
  per GPU, bf16 + fp32 master weights, AdamW; a step = forward + loss +
  tcgen05 backward + ONE all-reduce of [gradient | loss, counts] (NCCL under
  torchrun) + update, timed with CUDA events, max over ranks.
* ``config4`` (side line, N=1): BASELINE config 4's density sweep with the
  cuDNN dense-conv crossover comparator.
* ``interleave`` (side line, N=1): north_star (1)'s standalone kernels, GB/s.
* ``froxelize`` / ``gt_pvs`` (side lines, N=1): SURVEY §8(f) #1 / #3.

Multi-GPU: one process per GPU.  ``--gpus N`` with N > 1 outside torchrun
re-executes this script under ``torch.distributed.run`` with N ranks on
127.0.0.1; a WORLD_SIZE that disagrees with ``--gpus`` is an error.  Frames
are independent ("replicas only" per frame); value = total
frames / max-rank time.  ``--selftest`` runs the multi-rank plumbing on CPU
with gloo (the config-3 sharding over the numpy oracle), for the CPU tests.

``--impl reference`` times the CPU reference path (the oracle port) instead.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "froxel grids/sec and ms/frame (256^3, bs1); % tensor-pipe peak"
UNIT = "grids/s"
E2E_FRAMES = 64
E2E_INFLIGHT = 4  # frames computing concurrently in the streamed e2e (separate buffers per frame; tools/e2e_inflight.py: 3 -> 4 +1 %, 6 no better)
WORKLOAD = "config2: 256^3 froxels, 4000 boxes (edges 1-12, seed 1), d=4, 3-level sparse U-Net 64/128/256, bf16"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return p["hbm_gbs"], p["bf16_tflops"], "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.proc, self.lines = index, None, []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _free_port() -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def spawn(args) -> int:
    """Re-execute this script under torch.distributed.run with --gpus ranks (127.0.0.1)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def shard_range(n: int, rank: int, world: int):
    """Contiguous slice [r*n/N, (r+1)*n/N) of n independent units."""
    return rank * n // world, (rank + 1) * n // world


def run_selftest(args):
    """CPU / gloo check of the multi-rank plumbing: config-3 sharding (8 config-1
    grids through the numpy oracle at bs = slice), barrier-bracketed timing,
    max over ranks, one JSON line from rank 0 with a checksum of every grid's
    predicted bits (identical for any N)."""
    import hashlib

    import torch
    import torch.distributed as dist
    ws, rank, _ = dist_env()
    if ws > 1:
        dist.init_process_group("gloo")
    from oracle import sparse as osp
    from paper_2509_24677_b200 import synth
    G = 8
    lo, hi = shard_range(G, rank, ws)
    rng = np.random.Generator(np.random.PCG64(0))
    layers = []
    for k, cin, cout, act in ((3, 8, 32, "relu"), (3, 32, 32, "relu"), (1, 32, 8, "sigmoid")):
        w, b = osp.kaiming_uniform(rng, k ** 3, cin, cout, act)
        layers.append((k, w, b, act))
    occs = [synth.config3_grid(i) for i in range(lo, hi)]

    def step():
        out = []
        for occ in occs:
            cells = osp.interleave(occ.astype(np.float64), 2)[None]
            coords, prob = osp.chain_forward(cells, layers)
            dense = osp.deinterleave(osp.scatter_cells(coords, prob, (1,) + cells.shape[1:4])[0], 2)
            out.append(np.packbits((dense >= 0.5).transpose(2, 1, 0), axis=2, bitorder="little").tobytes())
        return out
    for _ in range(args.warmup):
        step()
    if ws > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        bits = step()
    dt = time.perf_counter() - t0
    if ws > 1:
        dist.barrier()
        t = torch.tensor([dt], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t[0])
        gathered = [None] * ws
        dist.all_gather_object(gathered, [hashlib.sha256(b).hexdigest() for b in bits])
        digests = sum(gathered, [])
    else:
        digests = [hashlib.sha256(b).hexdigest() for b in bits]
    if rank == 0:
        print(json.dumps({"impl": "selftest", "metric": "config3 sharding over the oracle (CPU, gloo)",
                          "value": G * args.steps / dt, "unit": "grids/s", "n_gpus": ws, "steps": args.steps,
                          "warmup": args.warmup, "grids": G, "shards": [list(shard_range(G, r, ws)) for r in range(ws)],
                          "checksum": hashlib.sha256("".join(digests).encode()).hexdigest()}), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def cpu_threads() -> int:
    """Give OpenBLAS every host thread (torchrun sets OMP_NUM_THREADS=1 per rank)."""
    n = os.cpu_count() or 1
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(n)
    except Exception:
        pass
    return n


def cpu_frame_time(occ, seed=1):
    """One config-2 frame through the numpy sparse restatement (oracle, float64)."""
    from oracle import sparse as osp
    params = osp.unet_init(seed)
    t0 = time.perf_counter()
    cells = osp.interleave(occ.astype(np.float64), 4)[None]
    coords, prob = osp.unet_forward(cells, params, bf16=False)
    dense = osp.deinterleave(osp.scatter_cells(coords, prob, (1,) + cells.shape[1:4])[0], 4)
    np.packbits((dense >= 0.5).transpose(2, 1, 0), axis=2, bitorder="little")
    return time.perf_counter() - t0


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    from paper_2509_24677_b200 import synth
    occ = synth.config2_grid(1)
    cores = cpu_threads()
    warm = min(args.warmup, 3)  # CPU frames take seconds; 3 covers the warm-up rule without stretching the run
    for _ in range(warm):
        cpu_frame_time(occ)
    times = [cpu_frame_time(occ) for _ in range(args.steps)]
    total = sum(times)
    value = args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": warm, "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded boxes; paper scenes unavailable)",
        "config": {"workload": WORKLOAD, "parallelism": "cpu, rank 0 only", "l2": "n/a (CPU)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": "one full config-2 frame per step: numpy sparse restatement of the reference "
                                   "arithmetic (oracle/sparse.py, float64, OpenBLAS on all host threads)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# number of our kernels each C-ABI entry point launches
KERNELS_PER_CALL = {"fpvs_kmap_compact": 1, "fpvs_hash_build": 1, "fpvs_levels_from_bits": 3, "fpvs_up_sort_multi": 2}


def count_launches(fn):
    """Run fn once while counting libfpvs kernel launches (via the C-ABI calls)."""
    from paper_2509_24677_b200 import _lib
    orig = _lib.call
    n = [0]

    def counting(name, *a):
        n[0] += KERNELS_PER_CALL.get(name, 1)
        return orig(name, *a)
    _lib.call = counting
    try:
        fn()
    finally:
        _lib.call = orig
    return n[0]


def train_config5(ws: int = 1, rank: int = 0, steps: int = 10, warmup: int = 3):
    """BASELINE config 5 per GPU: 8 grids of 128^3 (rank-specific seeds; weak
    scaling), config-1 net, bf16 compute with fp32 master weights, AdamW; a step
    = forward + fused loss + tcgen05 backward + ONE all-reduce of the
    [gradient | loss, counts] exchange buffer (NCCL over NVLink when N > 1) +
    update.  Device time with CUDA events, max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2509_24677_b200 import synth
    from paper_2509_24677_b200.froxel import FroxelGrid
    from paper_2509_24677_b200.neural import ModelConfig, PvsNet, TrainConfig
    from paper_2509_24677_b200.train import TrainStep
    B = 8
    pairs = [synth.config5_pair(rank, i) for i in range(B)]
    bits = torch.from_numpy(np.concatenate([FroxelGrid.from_dense(g).bits for g, _ in pairs])).cuda()
    # row LBL labels made on the device from the packed geometry (fpvs_first_hit_labels)
    gt = synth.first_hit_labels_bits(bits, B, (128, 128, 128), 2)
    want = torch.from_numpy(np.concatenate([FroxelGrid.from_dense(lb).bits for _, lb in pairs])).cuda()
    if not torch.equal(gt, want):
        raise RuntimeError("device labels differ from synth.first_hit_labels")
    net = PvsNet(ModelConfig.config1(), np.random.Generator(np.random.PCG64(0)), precision="bf16")
    step = TrainStep(net, B, (128, 128, 128), TrainConfig(optimizer="adamw", lr=1e-3))
    acc = torch.zeros(8, dtype=torch.float64, device="cuda")
    acc[6] = -1
    launches = {"allreduce": 0}
    if ws > 1:
        orig = dist.all_reduce

        def counting(*a, **k):
            launches["allreduce"] += 1
            return orig(*a, **k)
        dist.all_reduce = counting
    try:
        for i in range(warmup):
            step.forward_backward(bits, gt)
            step.exchange(1.0 / ws)
            step.accumulate(acc, i)
            step.update(1e-3, i + 1)
        torch.cuda.synchronize()
        launches["allreduce"] = 0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0.record()
        for i in range(steps):
            step.forward_backward(bits, gt)
            step.exchange(1.0 / ws)
            step.accumulate(acc, warmup + i)
            step.update(1e-3, warmup + i + 1)
        e1.record()
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
    finally:
        if ws > 1:
            dist.all_reduce = orig
    ms = e0.elapsed_time(e1) / steps
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t[0])
    a = acc.cpu().numpy()
    return {"workload": "config5: 8 x 128^3 grids per GPU, config-1 net, bf16 + fp32 master, AdamW lr 1e-3",
            "n_gpus": ws, "global_batch": B * ws, "scaling": "weak", "ms_per_step": ms,
            "grids_per_s": B * ws / (ms * 1e-3), "active_rows_rank0": step.lv.count(),
            "loss_mean": float(a[0] / max(a[1], 1)), "diverged": bool(a[6] >= 0),
            "allreduce_per_step": launches["allreduce"] / steps if ws > 1 else 0,
            "exchange_bytes": int(step.grads.numel() * 4), "backward": "tcgen05 dgrad + wgrad", "steps": steps}


def config3_line(ws: int = 1, rank: int = 0, steps: int = 20, warmup: int = 3, flush=None):
    """BASELINE config 3: 64 independent config-1 grids (seeds 100+i, density
    U(1%, 6%)) sharded contiguously over the ranks, each rank one batched frame
    of its slice per step (CUDA graph; L2 flushed between steps, untimed); no
    collective on the data path.  bf16 (tensor cores) and fp32 (SIMT, the
    config-1 parity precision).  grids/s = 64 * steps / max-rank time."""
    import torch
    import torch.distributed as dist
    from paper_2509_24677_b200 import synth
    from paper_2509_24677_b200.froxel import FroxelGrid
    from paper_2509_24677_b200.neural import ModelConfig, PvsNet
    from paper_2509_24677_b200.pipeline import FramePipeline
    G = 64
    lo, hi = shard_range(G, rank, ws)
    bits = torch.from_numpy(np.concatenate([FroxelGrid.from_dense(synth.config3_grid(i)).bits
                                            for i in range(lo, hi)])).cuda()
    out = {"workload": "config3: 64 x (64x64x32) grids, config-1 net, sharded [r*64/N, (r+1)*64/N)",
           "n_gpus": ws, "grids": G, "scaling": "strong", "slice_rank0": [lo, hi]}
    for prec in ("bf16", "fp32"):
        net = PvsNet(ModelConfig.config1(), np.random.Generator(np.random.PCG64(0)), precision=prec)
        pipe = FramePipeline(net, hi - lo, (64, 64, 32), graph=True)
        pipe.load(bits)
        pipe.capture()
        for _ in range(warmup):
            pipe.run_device()
        torch.cuda.synchronize()
        st = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        en = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for i in range(steps):
            if flush is not None:
                flush.zero_()
            st[i].record()
            pipe.run_device()
            en[i].record()
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        ms = sum(a.elapsed_time(b) for a, b in zip(st, en))
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        if ws > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0])
        out[prec] = {"grids_per_s": G * steps / (ms * 1e-3), "ms_per_batch": ms / steps,
                     "active_rows_rank0": pipe.plan.L0.count()}
    return out


def interleave_side(reps: int = 20):
    """North_star (1): the standalone interleave / deinterleave kernels at the
    config-2 size (256^3, d = 4) — algorithmic bytes (input + output, once) per
    call / device time, against the HBM peak.  Each timed call follows an
    untimed L2 flush; the call is replayed from a CUDA graph so the events
    bracket device work only."""
    import torch
    from paper_2509_24677_b200 import synth
    from paper_2509_24677_b200.froxel import FroxelGrid
    from paper_2509_24677_b200.interleave import deinterleave_device, interleave_device
    hbm, _, kind = peaks()
    occ = synth.config2_grid(1)
    dense = torch.from_numpy(occ.astype(np.float32)).cuda()[None]
    bits = torch.from_numpy(FroxelGrid.from_dense(occ).bits).cuda()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    dims = (1,) + occ.shape
    cells16 = interleave_device(dense, 4, torch.bfloat16)
    cells32 = interleave_device(dense, 4, torch.float32)
    cases = {
        "dense_f32_to_bf16": (lambda: interleave_device(dense, 4, torch.bfloat16), 4 * occ.size + 2 * occ.size),
        "packed_to_bf16": (lambda: interleave_device(bits, 4, torch.bfloat16, packed_dims=dims),
                           occ.size // 8 + 2 * occ.size),
        "deinterleave_f32_to_f32": (lambda: deinterleave_device(cells32, 4), 8 * occ.size),
        "deinterleave_bf16_threshold_bits": (lambda: deinterleave_device(cells16, 4, 0.5), 2 * occ.size + occ.size // 8),
    }
    out = {"workload": "256^3 froxels, d = 4 (config 2): 64^3 cells x 64 channels", "peak_gbs": hbm,
           "peak_kind": kind}
    from paper_2509_24677_b200.pipeline import no_gc

    def graph_of(body, k=8):
        g = torch.cuda.CUDAGraph()
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st), no_gc():
            with torch.cuda.graph(g, stream=st):
                for _ in range(k):
                    body()
        torch.cuda.current_stream().wait_stream(st)
        return g

    def timed(g):
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return statistics.median(ts)
    # per call: graphs of 8 x (L2 flush, call) and of 8 x (L2 flush) alone;
    # the difference / 8 is the call's device time with a cold L2 and no host
    # or graph-launch overhead inside
    k = 8
    t_flush = timed(graph_of(lambda: flush.zero_(), k))
    for name, (fn, nbytes) in cases.items():
        fn()
        torch.cuda.synchronize()
        g = graph_of(lambda fn=fn: (flush.zero_(), fn()), k)
        ms = max(timed(g) - t_flush, 1e-6) / k
        del g
        gbs = nbytes / (ms * 1e-3) / 1e9
        out[name] = {"us": round(ms * 1e3, 2), "bytes": int(nbytes), "gbs": round(gbs, 1), "frac": round(gbs / hbm, 3)}
    return out


def config4_line(flush, densities=(0.005, 0.02, 0.08, 0.25), reps: int = 10):
    """BASELINE config 4: the config-1 net (bf16) on 256^3 grids at swept
    occupancy — per-stage device time inside the L2-flushed frame
    (pipeline.frame_stage_times), HBM GB/s of the map stage and TFLOP/s of the
    convs — beside a DENSE comparator: the same network as cuDNN bf16 conv3d
    over the whole 128^3 x 8 interleaved grid (channels-last, the reference's
    dense semantics, torch.nn.functional.conv3d; used only as the crossover
    comparator, never on the product path).  ``crossover_density``: where the
    sparse frame time reaches the dense one (log-linear interpolation)."""
    import torch
    import torch.nn.functional as F
    from paper_2509_24677_b200 import synth
    from paper_2509_24677_b200.froxel import FroxelGrid
    from paper_2509_24677_b200.interleave import interleave_device
    from paper_2509_24677_b200.neural import ModelConfig, PvsNet
    from paper_2509_24677_b200.pipeline import FramePipeline, frame_stage_times, no_gc
    hbm, tf_peak, _ = peaks()
    net = PvsNet(ModelConfig.config1(), np.random.Generator(np.random.PCG64(0)), precision="bf16")
    torch.backends.cudnn.benchmark = True
    wts = []
    for L in net.layers:
        k, cin, cout = L.spec.kernel, L.spec.in_channels, L.spec.out_channels
        w = L.w.reshape(k, k, k, cin, cout).permute(4, 3, 0, 1, 2).contiguous().to(torch.bfloat16)
        wts.append((w.to(memory_format=torch.channels_last_3d), L.b.to(torch.bfloat16), k // 2, L.spec.activation))

    def dense_net(x):
        for w, b, pad, act in wts:
            x = F.conv3d(x, w, b, padding=pad)
            x = torch.relu_(x) if act == "relu" else torch.sigmoid(x)
        return x

    def timed_graph(body, captured=False):
        body()
        torch.cuda.synchronize()
        g = None
        if not captured:
            g = torch.cuda.CUDAGraph()
            st = torch.cuda.Stream()
            st.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(st), no_gc():
                with torch.cuda.graph(g, stream=st):
                    body()
            torch.cuda.current_stream().wait_stream(st)
        ts = []
        for _ in range(reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay() if g is not None else body()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        del g
        return statistics.median(ts)

    rows = []
    dense_ms = None
    for dens in densities:
        occ = synth.config4_grid(dens)
        bits = torch.from_numpy(FroxelGrid.from_dense(occ).bits).cuda()
        pipe = FramePipeline(net, 1, occ.shape, graph=True)
        pipe.load(bits)
        pipe.capture()
        frame = timed_graph(pipe.run_device, captured=True)
        stages, _ = frame_stage_times(pipe.plan, pipe.in_bits, pipe.out_bits, 0.5, flush=flush, reps=reps)
        n = pipe.plan.L0.count()
        lf = pipe.plan.layer_flops()
        conv_ms = sum(stages[k] for k in lf if k != "head")
        conv_fl = sum(v for k, v in lf.items() if k != "head")
        cells = pipe.plan.L0.ncells
        map_bytes = occ.size // 8 + 7 * cells + 124 * n + n * 8 * 2
        if dense_ms is None:
            x = interleave_device(bits, 2, torch.bfloat16, packed_dims=(1,) + occ.shape)  # (1, X, Y, Z, 8)
            xd = x.permute(0, 4, 1, 2, 3).contiguous(memory_format=torch.channels_last_3d)
            dense_ms = timed_graph(lambda: dense_net(xd))
            dense_flops = 2 * cells * sum(L.spec.kernel ** 3 * L.spec.in_channels * L.spec.out_channels
                                          for L in net.layers)
        rows.append({"density": float(occ.mean()), "target": dens, "active_cells": n, "cells": cells,
                     "frame_us": round(frame * 1e3, 1),
                     "maps_us": round(stages["maps"] * 1e3, 1),
                     "maps_gbs": round(map_bytes / (stages["maps"] * 1e-3) / 1e9, 1),
                     "maps_hbm_frac": round(map_bytes / (stages["maps"] * 1e-3) / 1e9 / hbm, 3),
                     "conv_us": round(conv_ms * 1e3, 1),
                     "conv_tflops": round(conv_fl / (conv_ms * 1e-3) / 1e12, 1),
                     "conv_tensor_frac": round(conv_fl / (conv_ms * 1e-3) / 1e12 / tf_peak, 3),
                     "head_us": round(stages["head"] * 1e3, 1),
                     "sparse_over_dense": round(frame / dense_ms, 3)})
    cross = None
    for a, b in zip(rows, rows[1:]):
        ra, rb = a["frame_us"] / (dense_ms * 1e3), b["frame_us"] / (dense_ms * 1e3)
        if ra < 1.0 <= rb:
            la, lb = np.log(a["density"]), np.log(b["density"])
            cross = float(np.exp(la + (np.log(1.0) - np.log(ra)) / (np.log(rb) - np.log(ra)) * (lb - la)))
    # sparse frame time is close to affine in the active-cell count: extrapolate
    # where it would reach the dense frame (as a fraction of all cells active)
    na = np.array([r["active_cells"] for r in rows], np.float64)
    fu = np.array([r["frame_us"] for r in rows], np.float64)
    slope, icpt = np.polyfit(na, fu, 1)
    n_star = (dense_ms * 1e3 - icpt) / slope if slope > 0 else float("inf")
    return {"workload": "config4: config-1 net (bf16) on 256^3 grids, d = 2 -> 128^3 cells",
            "crossover_active_fraction_extrapolated": round(float(n_star / rows[0]["cells"]), 3)
            if "cells" in rows[0] else None,
            "dense_comparator": "cuDNN bf16 conv3d (torch.nn.functional.conv3d, channels-last) over all 128^3 cells",
            "dense_frame_us": round(dense_ms * 1e3, 1),
            "dense_tflops": round(dense_flops / (dense_ms * 1e-3) / 1e12, 1), "sweep": rows,
            "crossover_density": cross if cross is not None else
            ("sparse faster at every swept density" if rows[-1]["sparse_over_dense"] < 1 else "dense faster at every swept density")}


def froxelize_side(reps: int = 20):
    """fpvs_froxelize of a seeded triangle scene into the 256^3
    grid (supersample 4, linear depth) — device time per call from a CUDA graph
    of ``reps`` calls; the oracle port (oracle/froxelize.py, numpy) on the same
    scene as its CPU baseline.  A reported side line, not the metric."""
    import torch
    from paper_2509_24677_b200 import synth
    from paper_2509_24677_b200.froxelize import FroxelizeConfig, Froxelizer, Frustum
    from oracle import froxelize as ofz
    dims = (256, 256, 256)
    out = {}
    for name, args, mode in (("scene0", (0, 12, 12), "perspective"), ("scene1", (1, 40, 24), "perspective"),
                             ("ortho_scene0", (0, 12, 12), "ortho"), ("ortho_scene1", (1, 40, 24), "ortho")):
        cfg = FroxelizeConfig(supersample=4, mode=mode)
        v, t, fa = synth.froxel_scene(*args)
        fr = Frustum.from_vectors(*fa)
        fz = Froxelizer(v, t)
        bits = torch.empty(256 ** 3 // 8, dtype=torch.uint8, device="cuda")
        fz.run(fr, dims, cfg, out=bits)
        torch.cuda.synchronize()
        samples = fz.samples()
        g = torch.cuda.CUDAGraph()
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        from paper_2509_24677_b200.pipeline import no_gc
        with torch.cuda.stream(st), no_gc():
            with torch.cuda.graph(g, stream=st):
                for _ in range(reps):
                    fz.run(fr, dims, cfg, out=bits)
        torch.cuda.current_stream().wait_stream(st)
        best = float("inf")
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) / reps)
        t0 = time.perf_counter()
        ref = (ofz.froxelize_ortho if mode == "ortho" else ofz.froxelize)(v, t, fr._o, fr._basis, fr.half_extent,
                                                                          fr.near, fr.far, dims, 4)
        cpu_s = time.perf_counter() - t0
        got = bits.cpu().numpy()
        out[name] = {"triangles": int(len(t)), "samples": int(samples), "device_us": round(best * 1e3, 2),
                     "gsamples_per_s": round(samples / (best * 1e-3) / 1e9, 2),
                     "oracle_cpu_s": round(cpu_s, 4), "speedup_vs_oracle": round(cpu_s / (best * 1e-3), 1),
                     "bit_exact_vs_oracle": bool(np.array_equal(got, ref))}
    return {"workload": "synth.froxel_scene -> 256^3 geometry grid, supersample 4, linear depth, viewcell frustum "
                        "(perspective and the dataset loop's three-view ortho mode)",
            "kernels": "setup + scan + raster (3 launches + memset)", **out}


def gt_pvs_side(views_n: int = 128):
    """fpvs_gt_pvs of a seeded scene for one viewcell — 128
    viewpoints (OracleConfig default), 1024^2 depth buffers, 256^3 grid — device
    time per viewcell (CUDA events, best of 3); the numpy oracle on ONE of the
    same viewpoints as its CPU baseline (per view).  A side line."""
    import torch
    from paper_2509_24677_b200 import gtpvs, synth, views
    from oracle import gtpvs as ogt
    dims = (256, 256, 256)
    v, t, fa = synth.froxel_scene(0, 12, 12)
    cell = views.ViewCell.from_forward(tuple(fa[0] + fa[5] * fa[1]), 0.3, 60.0, 15.0, tuple(fa[1]), 0.3, 20.0)
    ocfg = gtpvs.OracleConfig(viewpoints=views_n)
    g = gtpvs.GtPvs(v, t)
    out = torch.zeros(256 ** 3 // 8, dtype=torch.uint8, device="cuda")
    g.for_cell(cell, dims, ocfg, out=out)
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.for_cell(cell, dims, ocfg, out=out)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    cams = views.sample_viewpoints(cell, views_n)[:1]
    fr = views.build_viewcell_frustum(cell)
    t0 = time.perf_counter()
    ogt.gt_pvs(v, t, [c.params() for c in cams], (fr._o, fr._basis, fr.half_extent, fr.near, fr.far), dims,
               ocfg.resolution_for(dims))
    cpu_view_s = time.perf_counter() - t0
    return {"workload": f"synth.froxel_scene(0): {len(t)} triangles, {views_n} viewpoints, 1024x1024 depth buffers, "
                        "256^3 GT grid, linear depth",
            "kernels": "setup + scan + depth (64-bit atomicMin z-test) + resolve (4 launches + 2 memsets)",
            "device_ms_per_viewcell": round(best, 3), "device_us_per_view": round(best * 1e3 / views_n, 2),
            "gt_froxels": int(np.unpackbits(out.cpu().numpy()).sum()),
            "oracle_cpu_s_per_view": round(cpu_view_s, 4),
            "speedup_vs_oracle": round(cpu_view_s * views_n / (best * 1e-3), 1)}


def single_frame_latency(pipe, host_ins, host_out, frames: int = 20):
    """bs1 end to end with ONE frame in flight: pinned host packed grid -> H2D ->
    frame (graph replay) -> D2H packed PVS -> synchronise, per frame.  Device
    time between events before the upload and after the download, plus the
    host wall time of the same span; medians over ``frames``."""
    import torch
    dev, wall = [], []
    stream = torch.cuda.current_stream()
    for i in range(frames):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        e0.record(stream)
        pipe.in_bits.copy_(host_ins[i % len(host_ins)], non_blocking=True)
        pipe.run_device()
        host_out.copy_(pipe.out_bits, non_blocking=True)
        e1.record(stream)
        e1.synchronize()
        wall.append(time.perf_counter() - w0)
        dev.append(e0.elapsed_time(e1))
    return {"frames_in_flight": 1, "device_ms": statistics.median(dev), "wall_ms": 1e3 * statistics.median(wall),
            "frames": frames}


def run_ours(args):
    import torch
    import torch.distributed as dist
    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2509_24677_b200 import synth
    from paper_2509_24677_b200.froxel import FroxelGrid
    from paper_2509_24677_b200.pipeline import FramePipeline, frame_stage_times
    from paper_2509_24677_b200.unet import PvsUNet

    dims = (256, 256, 256)
    occ = synth.config2_grid(1)
    host_bits = torch.from_numpy(FroxelGrid.from_dense(occ).bits).pin_memory()
    nbytes = host_bits.numel()
    net = PvsUNet(seed=1, precision="bf16")
    pipe = FramePipeline(net, 1, dims, tau=0.5, graph=True)
    pipe.load(host_bits.cuda())
    pipe.capture()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()

    # ---- per-stage device times inside the L2-flushed frame, FLOPs, launch count
    layer_flops = pipe.plan.layer_flops()
    n0, n1, n2 = pipe.plan.counts()
    launches_per_frame = count_launches(lambda: pipe.plan.run(pipe.in_bits, pipe.out_bits, 0.5))
    torch.cuda.synchronize()
    stage_dev, staged_frame_ms = frame_stage_times(pipe.plan, pipe.in_bits, pipe.out_bits, 0.5, flush=flush, reps=20)
    conv_ms = {k: stage_dev[k] for k in layer_flops if k != "head"}
    head_fused = "head" not in stage_dev
    if head_fused:  # the head runs inside dec0b's launch: its FLOPs count there
        layer_flops = dict(layer_flops)
        layer_flops["dec0b"] += layer_flops.pop("head")
    pipe.capture(tune=False)  # the timed graph (no stage events)

    # ---- warm-up graph replays
    for _ in range(args.warmup):
        flush.zero_()
        pipe.run_device()
    torch.cuda.synchronize()

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    # ---- timed: device-resident input, graph replay per step
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for i in range(args.steps):
        flush.zero_()
        starts[i].record(stream)
        pipe.run_device()
        ends[i].record(stream)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    dev_ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))

    # ---- timed e2e: pinned host in -> device -> pinned host out, every step,
    # through the streaming API (frame i's compute overlaps frame i+1's upload
    # and frame i-1's download; every frame's copies are inside the region)
    # 64 distinct input frames (the config-2 scene shifted by whole cells:
    # same density), 128 MiB in total > the 126 MB L2, cycled over the steps
    host_ins = [host_bits]
    for k in range(1, E2E_FRAMES):
        shifted = np.roll(occ, (8 * (k % 8), 8 * (k // 8), 0), axis=(0, 1, 2))
        host_ins.append(torch.from_numpy(FroxelGrid.from_dense(shifted).bits).pin_memory())
    host_outs = [torch.empty(nbytes, dtype=torch.uint8, pin_memory=True) for _ in range(args.steps)]
    pipe.infer_stream([host_ins[i % 2] for i in range(4)], host_outs[:4], inflight=E2E_INFLIGHT)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    wall0 = time.perf_counter()
    e0.record(stream)
    pipe.infer_stream([host_ins[i % E2E_FRAMES] for i in range(args.steps)], host_outs, inflight=E2E_INFLIGHT)
    e1.record(stream)
    torch.cuda.synchronize()
    wall_e2e = time.perf_counter() - wall0
    if ws > 1:
        dist.barrier()
    e2e_ms = e0.elapsed_time(e1)
    host_out = host_outs[-1]
    latency = single_frame_latency(pipe, host_ins, torch.empty(nbytes, dtype=torch.uint8, pin_memory=True))
    time.sleep(0.2)
    clocks = sampler.stop()

    # correctness guard: the timed output equals the eager output
    pipe.in_bits.copy_(host_bits.cuda())
    pipe.run_device()
    check = pipe.out_bits.clone()
    pipe.plan.run(pipe.in_bits, pipe.out_bits, 0.5)
    torch.cuda.synchronize()
    if not torch.equal(check, pipe.out_bits):
        raise RuntimeError("graph replay output differs from the eager frame")
    # the streamed output of the last step equals an eager frame of the same input
    last_in = host_ins[(args.steps - 1) % E2E_FRAMES].cuda()
    pipe.plan.run(last_in, pipe.out_bits, 0.5)
    torch.cuda.synchronize()
    if not torch.equal(host_out.cuda(), pipe.out_bits):
        raise RuntimeError("streamed e2e output differs from the eager frame")

    t = torch.tensor([dev_ms, e2e_ms, latency["device_ms"], latency["wall_ms"]], dtype=torch.float64, device="cuda")
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dev_ms, e2e_ms = float(t[0]), float(t[1])
    latency["device_ms"], latency["wall_ms"] = float(t[2]), float(t[3])

    # ---- side lines at every N (collectives inside: all ranks take part)
    c3 = None if args.no_config3 else config3_line(ws, rank, steps=20, warmup=3, flush=flush)
    train = None if args.no_train else train_config5(ws, rank)
    if rank != 0:
        if ws > 1:
            dist.destroy_process_group()
        return 0

    hbm_peak, tf_peak, peak_kind = peaks()
    tc_ms = sum(conv_ms.values())
    tc_flops = sum(layer_flops[k] for k in conv_ms)
    # (a stage can difference to 0 when timed under a profiler: no rate then)
    achieved = tc_flops / (tc_ms * 1e-3) / 1e12 if tc_ms > 0 else None
    n_tc_launches = len(conv_ms)
    per_layer = {k: {"ms": round(conv_ms[k], 5),
                     "tflops": round(layer_flops[k] / (conv_ms[k] * 1e-3) / 1e12, 2) if conv_ms[k] > 0 else None}
                 for k in conv_ms}
    stage_ms = {k: round(v, 5) for k, v in stage_dev.items()}
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            traffic = json.load(fh).get("conv_dram_bytes_per_launch")
    except Exception:
        pass

    cpu = None
    frox = None
    gtp = None
    il = None
    if ws == 1 and not args.no_froxelize:
        frox = froxelize_side()
        gtp = gt_pvs_side()
    c4 = None
    if ws == 1:
        il = interleave_side()
        if not args.no_config4:
            c4 = config4_line(flush)
    if ws == 1 and not args.no_cpu_baseline:
        cores = cpu_threads()
        t_cpu = cpu_frame_time(occ)
        cpu = {"value": 1.0 / t_cpu, "unit": UNIT, "cores": cores, "kind": "port",
               "sample": "one config-2 frame (interleave, maps, U-Net, threshold) through the numpy sparse "
                         "restatement oracle/sparse.py in float64 on all host threads (OpenBLAS)"}

    value = ws * args.steps / (dev_ms * 1e-3)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dev_ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic (seeded boxes; paper scenes unavailable)",
        "config": {"workload": WORKLOAD, "global_batch": ws, "grid": list(dims), "parallelism": f"replicas x{ws}",
                   "l2": "value: flushed before every step (256 MiB memset, untimed); e2e: 64 distinct input "
                         "frames (128 MiB > L2) cycled, no flush",
                   "active_cells": [n0, n1, n2], "density": float(occ.mean()), "cuda_graph": True},
        "e2e": {"value": ws * args.steps / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": nbytes,
                "d2h_bytes_per_step": nbytes, "ms_per_step": e2e_ms / args.steps,
                "wall_ms_per_step": 1e3 * wall_e2e / args.steps, "frames_in_flight": E2E_INFLIGHT,
                "latency_ms": latency},
        "roofline": {"bound": "tensor",
                     "kernel": "tcgen05 sparse conv: spconv_halo (10 subm convs, halo-cached, A in TMEM; the 1x1x1 "
                               "head fused into dec0b's epilogue) + spconv_tc (2 down gather-GEMMs + 2 column-block up GEMMs) "
                               "per frame",
                     "head_fused": head_fused,
                     "achieved": achieved, "peak": tf_peak, "unit": "TFLOP/s",
                     "frac": achieved / tf_peak if achieved is not None else None,
                     "peak_kind": f"{peak_kind} bf16 burst", "traffic": traffic,
                     "traffic_unit": "DRAM bytes per launch (mean over the 14 conv launches, ncu --set full)",
                     "flops_per_frame": tc_flops, "launches_per_frame": n_tc_launches,
                     "kernel_ms_per_frame": tc_ms, "per_layer": per_layer,
                     "timing": "per stage inside the L2-flushed frame: prefix graphs of the frame's first k stages, "
                               "stage k = T_k - T_(k-1), medians of 20 replays (pipeline.frame_stage_times)"},
        "stages_ms": stage_ms,
        "stages_total_ms": round(sum(stage_dev.values()), 5),
        "staged_frame_ms": round(staged_frame_ms, 5),
        "gpu_launches": launches_per_frame * args.steps,
        "clocks": clocks,
    }
    if cpu is not None:
        line["cpu_baseline"] = cpu
    if c3 is not None:
        line["config3"] = c3
    if train is not None:
        line["train_config5"] = train
    if il is not None:
        line["interleave"] = il
    if c4 is not None:
        line["config4"] = c4
    if frox is not None:
        line["froxelize"] = frox
    if gtp is not None:
        line["gt_pvs"] = gtp
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-train", action="store_true", help="skip the config-5 training-step line")
    ap.add_argument("--no-config3", action="store_true", help="skip the config-3 sharded-batch line")
    ap.add_argument("--no-config4", action="store_true", help="skip the config-4 density sweep / dense crossover line")
    ap.add_argument("--no-froxelize", action="store_true", help="skip the froxelization / GT-PVS side lines")
    ap.add_argument("--selftest", action="store_true", help="CPU/gloo check of the multi-rank plumbing")
    args = ap.parse_args()
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return spawn(args)
    ws, _, _ = dist_env()
    if ws != args.gpus:
        print(f"bench.py: WORLD_SIZE={ws} but --gpus {args.gpus}", file=sys.stderr)
        return 2
    if args.selftest:
        return run_selftest(args)
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
