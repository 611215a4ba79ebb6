"""Streamed end-to-end throughput with B grids per launch chain (a lane runs
one B-grid frame plan; host buffers hold B packed grids), against frames in
flight — whether batching frames inside a lane beats more lanes of one
frame each.  Reported in grids/s (B grids per step)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_24677_b200 import synth  # noqa: E402
from paper_2509_24677_b200.froxel import FroxelGrid  # noqa: E402
from paper_2509_24677_b200.pipeline import FramePipeline  # noqa: E402
from paper_2509_24677_b200.unet import PvsUNet  # noqa: E402

occ = synth.config2_grid(1)
grids = []
for k in range(16):
    shifted = np.roll(occ, (8 * (k % 8), 8 * (k // 8), 0), axis=(0, 1, 2))
    grids.append(FroxelGrid.from_dense(shifted).bits)
steps = int(os.environ.get("STEPS", "32"))
for B in [int(v) for v in os.environ.get("BATCH", "1,2,4").split(",")]:
    host_ins = [torch.from_numpy(np.concatenate([grids[(s * B + j) % 16] for j in range(B)])).pin_memory()
                for s in range(8)]
    host_outs = [torch.empty(host_ins[0].numel(), dtype=torch.uint8, pin_memory=True) for _ in range(steps)]
    pipe = FramePipeline(PvsUNet(seed=1), B, occ.shape, graph=True)
    pipe.load(host_ins[0].cuda())
    pipe.capture()
    for inflight in [int(v) for v in os.environ.get("INFLIGHT", "1,2,4").split(",")]:
        pipe.infer_stream([host_ins[i % 8] for i in range(2 * inflight)], host_outs[:2 * inflight], inflight=inflight)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            pipe.infer_stream([host_ins[i % 8] for i in range(steps)], host_outs, inflight=inflight)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) / steps)
        print(f"B {B} inflight {inflight}: {best * 1e3:7.1f} us/step = {B * 1e3 / best:7.0f} grids/s", flush=True)
    del pipe
