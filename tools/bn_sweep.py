"""Device time of the down/up convs of the config-2 frame over tile widths bn."""
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
print("auto bn", {k: v for k, v in plan.bn.items() if k.startswith(("down", "up"))}, flush=True)
base = dict(plan.bn)
for name in ("down01", "down12", "up21", "up10"):
    for bn in (32, 64, 128, 256):
        cout = plan.net.layers[name].spec.out_channels
        if bn > 256 or bn > max(cout, 32) * 2:
            continue
        plan.bn = dict(base)
        plan.bn[name] = bn
        try:
            plan.run(bits, out, 0.5)
            torch.cuda.synchronize()
            t = device_stage_times(plan, bits, out, flush=flush)
            print(f"{name} bn={bn}: {t[name] * 1000:.2f} us", flush=True)
        except Exception as e:  # noqa: BLE001
            print(f"{name} bn={bn}: {type(e).__name__} {e}", flush=True)
plan.bn = base
