"""Per-phase timestamps of the tcgen05 kernel for CTA 0 (FPVS_TC_DEBUG=16)."""
import ctypes
import os
import sys

os.environ["FPVS_TC_DEBUG"] = str(16 | int(os.environ.get("EXTRA", "0")))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_24677_b200 import _lib, synth  # noqa: E402
from paper_2509_24677_b200.froxel import FroxelGrid  # noqa: E402
from paper_2509_24677_b200.neural import run_conv  # noqa: E402
from paper_2509_24677_b200.unet import PvsUNet  # noqa: E402

occ = synth.config2_grid(1)
bits = torch.from_numpy(FroxelGrid.from_dense(occ).bits).cuda()
net = PvsUNet(seed=1, precision="bf16")
plan = net.plan(1, occ.shape)
out = torch.empty(occ.size // 8, dtype=torch.uint8, device="cuda")
plan.run(bits, out, 0.5)
L0 = plan.L0
lib = _lib.load()
fn = lib.fpvs_debug_tc_timestamps
for name in ("enc0a", "enc0b", "head"):
    for _ in range(2):
        if name == "head":
            from paper_2509_24677_b200.neural import run_head
            run_head(net.layers["head"], plan.t0b, 64, L0, 4, occ.shape, 0.5, out, None, None, "bf16")
        else:
            x = plan.x0 if name == "enc0a" else plan.t0a
            run_conv(net.layers[name], x, 64, L0.nbr, 27, L0.n, L0.cap, plan.t0b, 64, 0, "bf16", act="relu")
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * 8192)()
    fn(buf, 8192)
    ts = np.array(buf[:4096], dtype=np.int64)
    t0 = ts[0]
    rel = lambda i: (ts[i] - t0) / 1000.0 if ts[i] >= t0 else float("nan")  # noqa: E731
    print(name, "setup %.2f us, end %.2f, after-sync %.2f" % (rel(1), rel(2), rel(3)))
    for t in range(4):
        b = 8 + 8 * t
        print("  tile %d: prod start %.2f maps %.2f issued %.2f | mma first %.2f last %.2f | epi start %.2f done %.2f"
              % (t, rel(b), rel(b + 1), rel(b + 2), rel(b + 3), rel(b + 4), rel(b + 5), rel(b + 6)))
# per-stage detail of the last run (head), then re-run enc0a for detail
run_conv(net.layers["enc0a"], plan.x0, 64, L0.nbr, 27, L0.n, L0.cap, plan.t0b, 64, 0, "bf16", act="relu")
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 8192)()
fn(buf, 8192)
ts = np.array(buf[:4096], dtype=np.int64)
t0 = ts[0]
print("chunk: A-empty-ok A-arrived | B-empty-ok | MMA-full-ok MMA-commit  (us)")
for k in list(range(0, 30)) + list(range(200, 215)):
    f = lambda i: (ts[i] - t0) / 1000.0  # noqa: E731
    print(k, "%.2f %.2f | %.2f %.2f" % (f(200 + k), f(600 + k), f(1000 + k), f(1400 + k)))
