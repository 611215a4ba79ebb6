"""Per-CTA phase times of the dense-brick conv (profiling build, globaltimer):
kernel start -> PDL wait done -> first halo chunk landed -> first MMA ->
last commit -> epilogue start -> epilogue end, for LAYER (default enc2a) of
the config-2 frame run alone (L2 warm)."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("FPVS_LIB", os.path.join(ROOT, "paper_2509_24677_b200", "libfpvs_prof.so"))
os.environ.setdefault("FPVS_BRICK", "2")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_24677_b200 import _lib, synth  # noqa: E402
from paper_2509_24677_b200.froxel import FroxelGrid  # noqa: E402
from paper_2509_24677_b200.unet import PvsUNet  # noqa: E402

occ = synth.config2_grid(1)
bits = torch.from_numpy(FroxelGrid.from_dense(occ).bits).cuda()
plan = PvsUNet(seed=1).plan(1, occ.shape)
plan.tune(bits)
out = torch.empty(occ.size // 8, dtype=torch.uint8, device="cuda")
plan.overlap = False
if os.environ.get("BRICK_LAYERS"):  # bricks only for these layers (the rest on the halo kernel)
    plan.set_bricks(plan.counts(), {k: plan.brick_cfg for k in os.environ["BRICK_LAYERS"].split(",")})
plan.run(bits, out, 0.5)
torch.cuda.synchronize()
stages = dict(plan.stages(bits, out, 0.5))
name = os.environ.get("LAYER", "enc2a")
print("brick cfg", plan.brick_of.get(name))
lib = _lib.load()
buf = (ctypes.c_ulonglong * (2 * 160 * 8))()
if os.environ.get("INFRAME"):
    # the frame's stages up to LAYER as one graph after an L2 flush (the
    # layer's real predecessors, programmatic launches and cache state)
    from paper_2509_24677_b200.pipeline import no_gc
    order = [n for n, _ in plan.stages(bits, out, 0.5)]
    pre = order[:order.index(name) + 1]
    lib.fpvs_debug_brick_reset_slot()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), no_gc():
        with torch.cuda.graph(g, stream=s):
            for n in pre:
                stages[n]()
            plan._join_side()
    torch.cuda.current_stream().wait_stream(s)
    flush = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        flush.zero_()
        g.replay()
        torch.cuda.synchronize()
else:
    for _ in range(3):
        ctypes.memset(buf, 0, ctypes.sizeof(buf))
        stages[name]()
        torch.cuda.synchronize()
lib.fpvs_debug_brick_times(buf)
clk = (ctypes.c_longlong * (2 * 160 * 8))()
lib.fpvs_debug_brick_clocks(clk)
# in-frame: the brick launches of the captured prefix alternate slots 0, 1 (capture order);
# SLOT picks one (default: the last brick launch of the prefix)
allt = np.frombuffer(buf, dtype=np.uint64).reshape(2, 160, 8).astype(np.int64)
allc = np.frombuffer(clk, dtype=np.int64).reshape(2, 160, 8)
slot = int(os.environ.get("SLOT", "-1"))
if slot < 0:
    slot = int(np.argmax([allt[k, :, 0].max() for k in (0, 1)]))
t, ck = allt[slot], allc[slot]
if (allt[0, :, 0] > 0).any() and (allt[1, :, 0] > 0).any():
    a, b = (allt[0], allt[1]) if allt[0, :, 0].max() < allt[1, :, 0].max() else (allt[1], allt[0])
    a, b = a[a[:, 0] > 0], b[b[:, 0] > 0]
    print("two launches: first ends (last epilogue) %.2f us before the second's first CTA start; "
          "second's data wait ends %.2f us after the first's end; second's first MMA %.2f us after" % (
              (b[:, 0].min() - a[:, 6].max()) / -1e3, (np.median(b[:, 1]) - a[:, 6].max()) / 1e3,
              (np.median(b[:, 3]) - a[:, 6].max()) / 1e3))
ok = t[:, 0] > 0
t = t[ok]
ck = ck[ok]
for k in range(0, len(t), 32):
    print("CTA %3d: mma0 %.2f chunk0 %.2f commit %.2f us | cycles mma0->chunk0 %d, chunk0->commit %d" % (
        k, (t[k, 3] - t[:, 0].min()) / 1e3, (t[k, 7] - t[:, 0].min()) / 1e3, (t[k, 4] - t[:, 0].min()) / 1e3,
        ck[k, 7] - ck[k, 3], ck[k, 4] - ck[k, 7]))
mma = (ck[:, 4] - ck[:, 3]).astype(np.float64)
print("MMA phase: %.0f SM cycles (median) over %.2f us -> %.0f MHz" % (
    np.median(mma), np.median(t[:, 4] - t[:, 3]) / 1e3, np.median(mma / ((t[:, 4] - t[:, 3]) / 1e3))))
t0 = t[:, 0].min()
labels = ["start", "data", "halo0", "mma0", "commit", "epi0", "epi1", "chunk0"]
print("CTAs", len(t), "| kernel span (first start -> last epilogue end) %.2f us" % ((t[:, 6].max() - t0) / 1e3))
for i, lab in enumerate(labels):
    v = (t[:, i] - t0) / 1e3
    print(f"{lab:7s} median {np.median(v):7.2f} us  min {v.min():7.2f}  max {v.max():7.2f}")
