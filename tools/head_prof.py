import os, sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2509_24677_b200 import synth
from paper_2509_24677_b200.froxel import FroxelGrid
from paper_2509_24677_b200.unet import PvsUNet
occ = synth.config2_grid(1)
bits = torch.from_numpy(FroxelGrid.from_dense(occ).bits).cuda()
plan = PvsUNet(seed=1).plan(1, occ.shape)
plan.tune(bits)
out = torch.empty(occ.size // 8, dtype=torch.uint8, device="cuda")
plan.run(bits, out, 0.5)
torch.cuda.synchronize()
stages = dict(plan.stages(bits, out, 0.5))
torch.cuda.cudart().cudaProfilerStart()
stages["head"]()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
