"""Per-layer output-tile width sweep on the cfg2 frame (device stage times)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2509_24677_b200 import synth  # noqa: E402
from paper_2509_24677_b200.froxel import FroxelGrid  # noqa: E402
from paper_2509_24677_b200.pipeline import device_stage_times  # noqa: E402
from paper_2509_24677_b200.unet import PvsUNet  # noqa: E402

occ = synth.config2_grid(1)
bits = torch.from_numpy(FroxelGrid.from_dense(occ).bits).cuda()
net = PvsUNet(seed=1, precision="bf16")
plan = net.plan(1, occ.shape)
out = torch.empty(occ.size // 8, dtype=torch.uint8, device="cuda")
plan.tune(bits)
base = dict(plan.bn)
print("tuned", base, plan.counts())
res = {}
for bn in (32, 64, 128, 256):
    plan.bn = {k: bn for k in base}
    plan.run(bits, out, 0.5)
    t = device_stage_times(plan, bits, out)
    res[bn] = t
    print(bn, {k: round(v * 1000, 1) for k, v in t.items() if k in base})
best = {k: min((res[b][k], b) for b in res) for k in base}
print("best", {k: (b, round(v * 1000, 1)) for k, (v, b) in best.items()})
