"""Per-layer device times of the config-2 halo convs over (bn, split) settings."""
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
out = torch.empty(occ.size // 8, dtype=torch.uint8, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
plan = net.plan(1, occ.shape)
plan.tune(bits)
base = dict(plan.halo_cfg)
print("auto", base, flush=True)
rows = {k: lv.count() for k, lv in plan.level_of.items()}
LAYERS = {0: ("enc0a", "dec0a"), 1: ("enc1a", "dec1a"), 2: ("enc2a",)}
CANDS = {0: [(64, -2), (64, 1), (64, -3), (64, -4), (64, 2)],
         1: [(128, 1), (128, 2), (128, 3), (128, 4), (128, -2), (64, 1), (64, 2)],
         2: [(128, 2), (128, 3), (128, 4), (128, 5), (64, 2), (64, 3), (256, 2), (256, 4)]}
for lvl, cands in CANDS.items():
    for c in cands:
        cfg = dict(base)
        for k in cfg:
            if k[-2] == str(lvl):
                cfg[k] = c
        plan.set_halo(rows, cfg)
        plan.run(bits, out, 0.5)
        torch.cuda.synchronize()
        t = device_stage_times(plan, bits, out, flush=flush)
        print(f"L{lvl} {c}: " + " ".join(f"{k}={t[k] * 1000:.2f}" for k in LAYERS[lvl]) +
              f"   total {sum(t.values()) * 1000:.1f}", flush=True)
plan.set_halo(rows, base)
