import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2509_24677_b200 import synth
from paper_2509_24677_b200.froxel import FroxelGrid
from paper_2509_24677_b200.unet import PvsUNet
occ = synth.config2_grid(1)
bits = torch.from_numpy(FroxelGrid.from_dense(occ).bits).cuda()
net = PvsUNet(seed=1)
for cfg in [None, {"enc0a": (64, 1), "enc0b": (64, 1), "dec0a": (64, 1), "dec0b": (64, 1)}, "tune"]:
    plan = net.plan(1, occ.shape)
    if cfg == "tune":
        plan.tune(bits)
    elif cfg:
        rows = {k: lv.cap for k, lv in plan.level_of.items()}
        plan.set_halo(rows, cfg)
    logits = torch.zeros((plan.L0.cap, 64), device="cuda")
    out = torch.empty(occ.size // 8, dtype=torch.uint8, device="cuda")
    acts = {}
    plan.run(bits, out, 0.5, logits=logits)
    torch.cuda.synchronize()
    n = plan.L0.count()
    bad = {name: bool(torch.isnan(getattr(plan, b)[:c].float()).any()) for name, b, c in
           [("t0a", "t0a", n), ("t0b", "t0b", n), ("buf0", "buf0", n), ("t1a", "t1a", plan.L1.count()), ("buf1", "buf1", plan.L1.count()), ("t2a", "t2a", plan.L2.count())]}
    print(cfg if cfg is None or cfg == "tune" else "L0 s1", plan.halo_cfg, "nan logits", bool(torch.isnan(logits[:n]).any()), bad)
