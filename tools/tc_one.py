"""Run a few config-2 enc0a launches (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2509_24677_b200 import synth  # noqa: E402
from paper_2509_24677_b200.froxel import FroxelGrid  # noqa: E402
from paper_2509_24677_b200.neural import run_conv  # noqa: E402
from paper_2509_24677_b200.unet import PvsUNet  # noqa: E402

occ = synth.config2_grid(1)
bits = torch.from_numpy(FroxelGrid.from_dense(occ).bits).cuda()
net = PvsUNet(seed=1, precision="bf16")
plan = net.plan(1, occ.shape)
out = torch.empty(occ.size // 8, dtype=torch.uint8, device="cuda")
plan.run(bits, out, 0.5)
L0 = plan.L0
for _ in range(3):
    run_conv(net.layers["enc0a"], plan.x0, 64, L0.nbr, 27, L0.n, L0.cap, plan.t0b, 64, 0, "bf16", act="relu")
torch.cuda.synchronize()
print("ok")
