"""Fixed cost of one tcgen05 conv launch vs active rows (events, back-to-back launches)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_24677_b200 import sparse as sp  # noqa: E402
from paper_2509_24677_b200.neural import Conv3d, ConvSpec, run_conv, run_head  # noqa: E402

layer = Conv3d(ConvSpec(3, 64, 64, "relu"), np.random.default_rng(0), init="kaiming_uniform")
head = Conv3d(ConvSpec(1, 64, 64, "sigmoid"), np.random.default_rng(1), init="kaiming_uniform")
for dens in (0.0, 0.0005, 0.005, 0.05, 0.2):
    rng = np.random.default_rng(3)
    mask = rng.random((1, 64, 64, 64)) < dens
    lv = sp.new_level(1, (64, 64, 64))
    lv.active.copy_(torch.from_numpy(mask.reshape(-1).astype(np.uint8)).cuda())
    sp.compact(lv)
    sp.build_subm(lv)
    n = lv.count()
    x = torch.randn((lv.cap, 64), device="cuda").bfloat16()
    y = torch.empty_like(x)
    bits = torch.zeros(64 * 64 * 64 * 64 // 8, dtype=torch.uint8, device="cuda")
    res = []
    for name, fn in (("subm", lambda: run_conv(layer, x, 64, lv.nbr, 27, lv.n, lv.cap, y, 64, 0, "bf16")),
                     ("1x1", lambda: run_conv(head, x, 64, None, 1, lv.n, lv.cap, y, 64, 0, "bf16", act="relu"))):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            fn()
        e1.record()
        torch.cuda.synchronize()
        res.append((name, round(e0.elapsed_time(e1) / 50 * 1000, 1)))
    print(f"rows {n:7d} tiles {(n + 127) // 128:5d}", res)
