"""Time the halo-cached wgrad vs the gathering wgrad on the config-5 level (32 -> 32, 27 taps)."""
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
cin, cout = 32, 32
h = sp.build_halo(lv)
x = torch.randn((lv.cap, cin), device="cuda").bfloat16()
dz = torch.randn((lv.cap, cout), device="cuda").bfloat16()
dw = torch.empty((27 * cin, cout), device="cuda")
db = torch.empty(cout, device="cuda")
ws1 = torch.empty(_lib.size("fpvs_wgrad_tc_workspace_size", 27, cin, cout, lv.cap), dtype=torch.uint8, device="cuda")
ws2 = torch.empty(_lib.size("fpvs_wgrad_halo_workspace_size", lv.cap), dtype=torch.uint8, device="cuda")


def old():
    _lib.call("fpvs_spconv_wgrad_tc", _lib.ptr(x), cin, _lib.ptr(dz), cout, _lib.ptr(lv.nbr), 27, _lib.ptr(lv.n),
              lv.cap, cin, cout, _lib.ptr(dw), _lib.ptr(db), _lib.ptr(ws1), ws1.numel(), 0)


def new():
    _lib.call("fpvs_spconv_wgrad_halo", _lib.ptr(x), cin, _lib.ptr(dz), cout, _lib.ptr(lv.nbr), _lib.ptr(lv.n),
              lv.cap, _lib.ptr(h["rows"]), _lib.ptr(h["n"]), _lib.ptr(h["lnbr"]), cin, cout, _lib.ptr(dw),
              _lib.ptr(db), _lib.ptr(ws2), ws2.numel(), 0)


flops = 2 * int((lv.nbr[:n] >= 0).sum()) * cin * cout
hn = h["n"][: (n + 127) // 128].float()
print(f"rows {n}, halo rows per tile mean {hn.mean():.0f} max {hn.max():.0f}")
for name, fn in (("gather", old), ("halo", new)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{name:7s} wgrad {ms * 1000:.1f} us  {flops / ms / 1e9:.1f} TFLOP/s", flush=True)
