"""Config-5 training step timing (8 x 128^3 grids, config-1 net, bf16 / fp32)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_24677_b200 import synth  # noqa: E402
from paper_2509_24677_b200.froxel import FroxelGrid  # noqa: E402
from paper_2509_24677_b200.neural import ModelConfig, PvsNet, TrainConfig  # noqa: E402
from paper_2509_24677_b200.train import TrainStep  # noqa: E402

B = int(os.environ.get("B", "8"))
pairs = [synth.config5_pair(0, i) for i in range(B)]
bits = torch.from_numpy(np.concatenate([FroxelGrid.from_dense(g).bits for g, _ in pairs])).cuda()
gt = torch.from_numpy(np.concatenate([FroxelGrid.from_dense(l).bits for _, l in pairs])).cuda()
for prec in os.environ.get("PREC", "bf16,fp32").split(","):
    net = PvsNet(ModelConfig.config1(), np.random.Generator(np.random.PCG64(0)), precision=prec)
    tcfg = TrainConfig(optimizer="adamw", lr=1e-3)
    step = TrainStep(net, B, (128, 128, 128), tcfg)
    for i in range(3):
        step.forward_backward(bits, gt)
        step.update(1e-3, i + 1)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    n = 10
    ev[0].record()
    for i in range(n):
        step.forward_backward(bits, gt)
        step.update(1e-3, 4 + i)
    ev[1].record()
    torch.cuda.synchronize()
    # forward only / backward only split
    ev[2].record()
    for i in range(n):
        step.backward()
    ev[3].record()
    torch.cuda.synchronize()
    rows = step.lv.count()
    print(f"{prec}: rows {rows}, step {ev[0].elapsed_time(ev[1]) / n:.3f} ms, backward alone "
          f"{ev[2].elapsed_time(ev[3]) / n:.3f} ms, loss {float(step.loss):.5f}", flush=True)
