"""Time fpvs_spconv_wgrad_tc on a config-5-sized level (profiling aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_24677_b200 import _lib, sparse as sp, synth  # noqa: E402
from paper_2509_24677_b200.froxel import FroxelGrid  # noqa: E402

grids = [synth.config5_pair(0, i)[0] for i in range(8)]
bits = torch.from_numpy(np.concatenate([FroxelGrid.from_dense(g).bits for g in grids])).cuda()
lv = sp.level_from_bits(bits, 8, (128, 128, 128), 2)
n = lv.count()
K, cin, cout = 27, int(os.environ.get("CIN", "32")), 32
x = torch.randn((lv.cap, cin), device="cuda").bfloat16()
dz = torch.randn((lv.cap, cout), device="cuda").bfloat16()
dw = torch.empty((K * cin, cout), device="cuda")
db = torch.empty(cout, device="cuda")
ws = torch.empty(_lib.size("fpvs_wgrad_tc_workspace_size", K, cin, cout, lv.cap), dtype=torch.uint8, device="cuda")


def run():
    _lib.call("fpvs_spconv_wgrad_tc", _lib.ptr(x), cin, _lib.ptr(dz), cout, _lib.ptr(lv.nbr), K, _lib.ptr(lv.n), lv.cap,
              cin, cout, _lib.ptr(dw), _lib.ptr(db), _lib.ptr(ws), ws.numel(), 0)


for _ in range(3):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    run()
e1.record()
torch.cuda.synchronize()
flops = 2 * int((lv.nbr[:n] >= 0).sum()) * cin * cout
ms = e0.elapsed_time(e1) / 10
print(f"dbg={os.environ.get('FPVS_WGRAD_DEBUG', '0')} rows {n} wgrad {ms * 1000:.1f} us  {flops / ms / 1e9:.1f} TFLOP/s")

if int(os.environ.get("FPVS_WGRAD_DEBUG", "0")) & 32:
    import ctypes
    buf = (ctypes.c_ulonglong * 4096)()
    _lib.load().fpvs_debug_wgrad_timestamps(buf)
    tt = np.frombuffer(buf, dtype=np.uint64).astype(np.int64).reshape(512, 8)
    t0 = tt[0, 0]
    for k in range(min(20, 512)):
        if tt[k, 0] == 0:
            break
        print(k, " ".join(f"{(v - t0) / 1000:7.2f}" if v else "    nan" for v in tt[k, :6]))
