"""Time one config-2 layer shape on the tcgen05 kernel (profiling aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_24677_b200 import synth  # noqa: E402
from paper_2509_24677_b200.froxel import FroxelGrid  # noqa: E402
from paper_2509_24677_b200.unet import PvsUNet  # noqa: E402

occ = synth.config2_grid(1)
bits = torch.from_numpy(FroxelGrid.from_dense(occ).bits).cuda()
net = PvsUNet(seed=1, precision="bf16")
plan = net.plan(1, occ.shape)
out = torch.empty(occ.size // 8, dtype=torch.uint8, device="cuda")
plan.tune(bits)
for _ in range(3):
    plan.run(bits, out, 0.5)
torch.cuda.synchronize()
from paper_2509_24677_b200.pipeline import stage_times  # noqa: E402
acc = {}
for _ in range(10):
    ev = []
    plan.run(bits, out, 0.5, events=ev)
    torch.cuda.synchronize()
    for k, v in stage_times(ev):
        acc.setdefault(k, []).append(v)
print(os.environ.get("FPVS_TC_DEBUG", "0"), {k: round(float(np.median(v)) * 1000, 1) for k, v in acc.items()})
