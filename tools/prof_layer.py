"""Run one conv stage of the config-2 frame a few times (for ncu -k regex:halo ... -c N)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2509_24677_b200 import synth  # noqa: E402
from paper_2509_24677_b200.froxel import FroxelGrid  # noqa: E402
from paper_2509_24677_b200.unet import PvsUNet  # noqa: E402

occ = synth.config2_grid(1)
bits = torch.from_numpy(FroxelGrid.from_dense(occ).bits).cuda()
plan = PvsUNet(seed=1).plan(1, occ.shape)
plan.tune(bits)
out = torch.empty(occ.size // 8, dtype=torch.uint8, device="cuda")
plan.overlap = False
plan.run(bits, out, 0.5)
torch.cuda.synchronize()
stages = dict(plan.stages(bits, out, 0.5))
for name in os.environ.get("LAYERS", "enc0b").split(","):
    for _ in range(int(os.environ.get("REPS", "2"))):
        stages[name]()
torch.cuda.synchronize()
print("ok")
