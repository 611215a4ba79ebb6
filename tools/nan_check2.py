import sys
sys.path.insert(0, '/root/repo')
sys.path.insert(0, '/root/repo/tests')
import numpy as np
import torch
from test_gpu_unet import _run, _check
from paper_2509_24677_b200 import synth
occ = synth.config2_grid(1)
plan, out, logits = _run(occ)
n = plan.L0.count()
lg = logits[:n].cpu().numpy()
print("nan rows", np.isnan(lg).any(1).sum(), "of", n, "first", np.nonzero(np.isnan(lg).any(1))[0][:10])
print("halo cfg", plan.halo_cfg)
err, hard, soft, vis = _check(occ, plan, out, logits)
print("err", err, hard, soft, vis)
