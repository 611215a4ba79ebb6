"""Per-stage device times of a config-2 frame (graph-replayed stages)."""
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
if os.environ.get("TUNE", "1") == "1":
    plan.tune(bits)
plan.run(bits, out, 0.5)
t = device_stage_times(plan, bits, out)
fl = plan.layer_flops()
tot = sum(t.values())
print(os.environ.get("FPVS_TC_VARIANT", "0"), "total %.1f us" % (tot * 1000))
print({k: round(v * 1000, 1) for k, v in t.items()})
print({k: round(fl[k] / (t[k] * 1e-3) / 1e12, 1) for k in fl})
