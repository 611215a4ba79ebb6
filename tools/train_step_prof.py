import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2509_24677_b200 import synth
from paper_2509_24677_b200.froxel import FroxelGrid
from paper_2509_24677_b200.neural import ModelConfig, PvsNet, TrainConfig
from paper_2509_24677_b200.train import TrainStep
B = 8
pairs = [synth.config5_pair(0, i) for i in range(B)]
bits = torch.from_numpy(np.concatenate([FroxelGrid.from_dense(g).bits for g, _ in pairs])).cuda()
gt = torch.from_numpy(np.concatenate([FroxelGrid.from_dense(l).bits for _, l in pairs])).cuda()
net = PvsNet(ModelConfig.config1(), np.random.Generator(np.random.PCG64(0)), precision="bf16")
step = TrainStep(net, B, (128, 128, 128), TrainConfig(optimizer="adamw", lr=1e-3))
for i in range(3):
    step.forward_backward(bits, gt); step.update(1e-3, i + 1)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
step.forward_backward(bits, gt); step.update(1e-3, 9)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
