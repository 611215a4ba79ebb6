"""Run the cfg2 maps stage a few times (for an ncu launch list)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2509_24677_b200 import synth  # noqa: E402
from paper_2509_24677_b200.froxel import FroxelGrid  # noqa: E402
from paper_2509_24677_b200.unet import PvsUNet  # noqa: E402

occ = synth.config2_grid(1)
bits = torch.from_numpy(FroxelGrid.from_dense(occ).bits).cuda()
net = PvsUNet(seed=1, precision="bf16")
plan = net.plan(1, occ.shape)
for _ in range(3):
    plan.build_maps(bits)
torch.cuda.synchronize()
print("n", plan.L0.count(), plan.L1.count(), plan.L2.count())
