"""Streamed end-to-end throughput (pinned host grids in -> packed PVS out)
against the number of frames computing concurrently (bench.py's e2e leg)."""
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
steps = int(os.environ.get("STEPS", "60"))
host_ins = []
for k in range(64):
    shifted = np.roll(occ, (8 * (k % 8), 8 * (k // 8), 0), axis=(0, 1, 2))
    host_ins.append(torch.from_numpy(FroxelGrid.from_dense(shifted).bits).pin_memory())
nbytes = host_ins[0].numel()
host_outs = [torch.empty(nbytes, dtype=torch.uint8, pin_memory=True) for _ in range(steps)]
pipe = FramePipeline(PvsUNet(seed=1), 1, occ.shape, graph=True)
pipe.load(host_ins[0].cuda())
pipe.capture()
for inflight in [int(v) for v in os.environ.get("INFLIGHT", "1,2,3,4,6").split(",")]:
    pipe.infer_stream([host_ins[i % 2] for i in range(2 * inflight)], host_outs[:2 * inflight], inflight=inflight)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pipe.infer_stream([host_ins[i % 64] for i in range(steps)], host_outs, inflight=inflight)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / steps)
    print(f"inflight {inflight}: {best * 1e3:7.1f} us/frame = {1e3 / best:7.0f} grids/s")
