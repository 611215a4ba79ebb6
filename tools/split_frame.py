"""Whole-frame (graph replay after an L2 flush) device time over per-level
(bn, split) settings of the halo convs: the production library, the real
frame (tools/split_sweep.py timed layers alone)."""
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
bits = torch.from_numpy(FroxelGrid.from_dense(occ).bits).cuda()
flush = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
LV = {0: ("enc0a", "enc0b", "dec0a", "dec0b"), 1: ("enc1a", "enc1b", "dec1a", "dec1b"), 2: ("enc2a", "enc2b")}
CANDS = {1: [(128, 1), (128, 2), (64, 1), (64, 2), (128, -2)],
         2: [(128, 2), (128, 3), (128, 4), (64, 2), (64, 1), (256, 4)],
         0: [(64, 1), (64, -2), (64, -3)]}


def frame_us(cfg):
    pipe = FramePipeline(PvsUNet(seed=1), 1, occ.shape)
    pipe.load(bits)
    pipe.plan.tune(bits)
    rows = {k: lv.count() for k, lv in pipe.plan.level_of.items()}
    full = dict(pipe.plan.halo_cfg)
    full.update(cfg)
    if "dec0b" in cfg and cfg["dec0b"] != (64, 1):
        pass  # the fused head needs dec0b at (64, 1): the plan falls back to the stand-alone head
    pipe.plan.set_halo(rows, full)
    pipe.capture(tune=False)
    ts = []
    for _ in range(30):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pipe.run_device()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts)), dict(pipe.plan.halo_cfg)


base, auto = frame_us({})
print(f"auto {auto}: {base:.1f} us", flush=True)
for lvl in (1, 2, 0):
    for c in CANDS[lvl]:
        cfg = {k: c for k in LV[lvl] if not (k == "dec0b" and c != (64, 1))}
        t, _ = frame_us(cfg)
        print(f"level {lvl} {c}: {t:.1f} us ({t - base:+.1f})", flush=True)
