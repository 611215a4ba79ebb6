"""Config-5 training steps (bench.train_config5's loop, one GPU) for an ncu
launch list: which kernels a step spends its 0.7 ms in."""
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
gt = synth.first_hit_labels_bits(bits, B, (128, 128, 128), 2)
net = PvsNet(ModelConfig.config1(), np.random.Generator(np.random.PCG64(0)), precision="bf16")
step = TrainStep(net, B, (128, 128, 128), TrainConfig(optimizer="adamw", lr=1e-3))
acc = torch.zeros(8, dtype=torch.float64, device="cuda")
acc[6] = -1
for i in range(int(os.environ.get("STEPS", "3"))):
    step.forward_backward(bits, gt)
    step.exchange(1.0)
    step.accumulate(acc, i)
    step.update(1e-3, i + 1)
torch.cuda.synchronize()
print("ok")
