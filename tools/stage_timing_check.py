"""Compare per-stage timing methods for the config-2 frame (which one to trust).

(a) the frame as one graph with external timing events between stages,
(b) the frame launched eagerly with events between stages after a 1 GiB L2
    flush that keeps the GPU busy while the host enqueues the whole frame,
(c) each stage alone as a graph of 20 back-to-back launches (L2 warm).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_24677_b200 import synth  # noqa: E402
from paper_2509_24677_b200.froxel import FroxelGrid  # noqa: E402
from paper_2509_24677_b200.pipeline import FramePipeline, device_stage_times, frame_stage_times  # noqa: E402
from paper_2509_24677_b200.unet import PvsUNet  # noqa: E402

occ = synth.config2_grid(1)
pipe = FramePipeline(PvsUNet(seed=1), 1, occ.shape)
pipe.load(torch.from_numpy(FroxelGrid.from_dense(occ).bits).cuda())
pipe.capture()
flush = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
a, fa = frame_stage_times(pipe.plan, pipe.in_bits, pipe.out_bits, 0.5, flush=flush, reps=10)

stages = pipe.plan.stages(pipe.in_bits, pipe.out_bits, 0.5)
per = {n: [] for n, _ in stages}
frames = []
for _ in range(10):
    torch.cuda.synchronize()
    flush.zero_()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(len(stages) + 1)]
    for ev, (_, fn) in zip(evs, stages):
        ev.record()
        fn()
    evs[-1].record()
    torch.cuda.synchronize()
    for (n, _), e0, e1 in zip(stages, evs, evs[1:]):
        per[n].append(e0.elapsed_time(e1))
    frames.append(evs[0].elapsed_time(evs[-1]))
b = {k: float(np.median(v)) for k, v in per.items()}
c = device_stage_times(pipe.plan, pipe.in_bits, pipe.out_bits, 0.5, reps=20)
g = []
for _ in range(10):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    pipe.run_device()
    e1.record()
    torch.cuda.synchronize()
    g.append(e0.elapsed_time(e1))
print(f"graph frame (no events) {np.median(g) * 1e3:.1f} us | (a) sum {sum(a.values()) * 1e3:.1f} frame {fa * 1e3:.1f}"
      f" | (b) sum {sum(b.values()) * 1e3:.1f} frame {np.median(frames) * 1e3:.1f} | (c) sum {sum(c.values()) * 1e3:.1f}")
for k in a:
    print(f"{k:8s} a {a[k] * 1e3:7.2f}  b {b[k] * 1e3:7.2f}  c {c[k] * 1e3:7.2f}")
