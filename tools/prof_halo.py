"""Two config-2 frames (halo kernel on); profiling target for ncu."""
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
cfg = os.environ.get("HALO_CFG")  # e.g. "64,1;128,1;128,1" per level
if cfg:
    per = [tuple(int(v) for v in c.split(",")) for c in cfg.split(";")]
    rows = {k: lv.count() for k, lv in plan.level_of.items()}
    lv_idx = {"0": 0, "1": 1, "2": 2}
    plan.set_halo(rows, {k: per[int(k[-2])] for k in rows})
out = torch.empty(occ.size // 8, dtype=torch.uint8, device="cuda")
for _ in range(2):
    plan.run(bits, out, 0.5)
torch.cuda.synchronize()
print("ok", plan.halo_cfg)
