"""Kernel-boundary cost inside the L2-flushed frame (profiling build): the
frame's stages up to LAYER as one graph, per-CTA spans of the last two halo
conv launches (per-launch slots): the second grid's first CTA start and its
loaders' data-ready (programmatic-launch wait done) against the first grid's
last CTA end.  LAYER=enc1b (pair enc1a -> enc1b) by default."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("FPVS_LIB", os.path.join(ROOT, "paper_2509_24677_b200", "libfpvs_prof.so"))
os.environ["FPVS_HALO_DEBUG"] = str(1 + 256 * 200)  # spans only: no CTA index 200, so no per-role stamps
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_24677_b200 import _lib, synth  # noqa: E402
from paper_2509_24677_b200.froxel import FroxelGrid  # noqa: E402
from paper_2509_24677_b200.pipeline import no_gc  # noqa: E402
from paper_2509_24677_b200.unet import PvsUNet  # noqa: E402

occ = synth.config2_grid(1)
bits = torch.from_numpy(FroxelGrid.from_dense(occ).bits).cuda()
plan = PvsUNet(seed=1).plan(1, occ.shape)
plan.tune(bits)
out = torch.empty(occ.size // 8, dtype=torch.uint8, device="cuda")
plan.overlap = False
plan.run(bits, out, 0.5)
torch.cuda.synchronize()
lib = _lib.load()
flush = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
for name in os.environ.get("LAYERS", "enc0b,enc1b,enc2b,dec1b,dec0b").split(","):
    stages = plan.stages(bits, out, 0.5)
    order = [n for n, _ in stages]
    fns = dict(stages)
    pre = order[:order.index(name) + 1]
    lib.fpvs_debug_halo_reset_slot.restype = ctypes.c_int
    lib.fpvs_debug_halo_reset_slot()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), no_gc():
        with torch.cuda.graph(g, stream=s):
            for n in pre:
                fns[n]()
            plan._join_side()
    torch.cuda.current_stream().wait_stream(s)
    nl = lib.fpvs_debug_halo_slot_count()  # halo launches in the captured prefix (slot = capture order)
    for _ in range(3):
        flush.zero_()
        torch.cuda.synchronize()
        lib.fpvs_debug_halo_reset_slot()  # clears the spans
        g.replay()
        torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (32 * 3 * 160))()
    lib.fpvs_debug_halo_cta_times(buf)
    sp = np.frombuffer(buf, dtype=np.uint64).astype(np.int64).reshape(32, 3, 160)
    a, b = sp[nl - 2], sp[nl - 1]
    ka, kb = a[0] > 0, b[0] > 0
    a_end = a[1][ka].max()
    print(f"{name}: previous halo grid ({ka.sum()} CTAs) last end -> this grid ({kb.sum()} CTAs): first CTA start "
          f"{(b[0][kb].min() - a_end) / 1e3:+.2f} us, median start {(np.median(b[0][kb]) - a_end) / 1e3:+.2f}, "
          f"data ready (loaders past the wait) median {(np.median(b[2][kb]) - a_end) / 1e3:+.2f} us; "
          f"previous grid's CTA ends spread {(a_end - a[1][ka].min()) / 1e3:.2f} us")
    del g
