"""One config-5 bf16 training step (ncu target)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_24677_b200 import synth  # noqa: E402
from paper_2509_24677_b200.froxel import FroxelGrid  # noqa: E402
from paper_2509_24677_b200.neural import ModelConfig, PvsNet, TrainConfig  # noqa: E402
from paper_2509_24677_b200.train import TrainStep  # noqa: E402

B = 8
pairs = [synth.config5_pair(0, i) for i in range(B)]
bits = torch.from_numpy(np.concatenate([FroxelGrid.from_dense(g).bits for g, _ in pairs])).cuda()
gt = torch.from_numpy(np.concatenate([FroxelGrid.from_dense(l).bits for _, l in pairs])).cuda()
net = PvsNet(ModelConfig.config1(), np.random.Generator(np.random.PCG64(0)), precision="bf16")
step = TrainStep(net, B, (128, 128, 128), TrainConfig(optimizer="adamw"))
for i in range(2):
    step.forward_backward(bits, gt)
    step.update(1e-3, i + 1)
torch.cuda.synchronize()
print("ok", float(step.loss))
