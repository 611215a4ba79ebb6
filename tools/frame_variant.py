"""Whole-frame device time (graph replay after an L2 flush, side streams on)
for environment variants of the U-Net plan: which optional stage pays off
inside the real frame.

  VARIANTS="base;FPVS_UPSORT=0;FPVS_FUSE_HEAD=0;overlap=0"   (';'-separated,
  each a ','-separated list of ENV=VAL; overlap=0 turns the side stream off)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_24677_b200 import synth  # noqa: E402
from paper_2509_24677_b200.froxel import FroxelGrid  # noqa: E402
from paper_2509_24677_b200.pipeline import FramePipeline  # noqa: E402
from paper_2509_24677_b200.unet import PvsUNet  # noqa: E402

variants = os.environ.get("VARIANTS", "base;FPVS_UPSORT=0;overlap=0").split(";")
reps = int(os.environ.get("REPS", "40"))
occ = synth.config2_grid(int(os.environ.get("SEED", "1")))
bits = torch.from_numpy(FroxelGrid.from_dense(occ).bits).cuda()
flush = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
ref = None
rows = []
for var in variants:
    saved = {}
    overlap = True
    for kv in var.split(","):
        if "=" not in kv:
            continue
        k, v = kv.split("=", 1)
        if k == "overlap":
            overlap = v != "0"
            continue
        saved[k] = os.environ.get(k)
        os.environ[k] = v
    pipe = FramePipeline(PvsUNet(seed=1), 1, occ.shape)
    pipe.plan.overlap = overlap
    pipe.load(bits)
    pipe.capture()
    pipe.run_device()
    torch.cuda.synchronize()
    out = pipe.out_bits.clone()
    if ref is None:
        ref = out
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pipe.run_device()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    rows.append((var, float(np.median(ts)), float(np.min(ts)), bool(torch.equal(out, ref))))
    for k, v in saved.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v
    del pipe
for var, med, mn, same in rows:
    print(f"{var:40s} frame {med:7.1f} us (min {mn:7.1f})  same bits as first: {same}")
