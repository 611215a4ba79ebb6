"""Which part of the compaction kernel K2 (levels.cu) costs its ~10 us in the
frame (profiling build; ablated results are wrong by construction): graphs of
K1 and of K1 + K2 (+ K3's look-back reset only, FPVS_LV_STOP) after an L2
flush, differenced, for each FPVS_K2_ABL bit set:
  1 no look-back, 2 no index_vol stores, 4 no coords stores, 8 no flag loads,
  16 no ticket atomic."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("FPVS_LIB", os.path.join(ROOT, "paper_2509_24677_b200", "libfpvs_prof.so"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_24677_b200 import synth  # noqa: E402
from paper_2509_24677_b200.froxel import FroxelGrid  # noqa: E402
from paper_2509_24677_b200.pipeline import no_gc  # noqa: E402
from paper_2509_24677_b200.unet import PvsUNet  # noqa: E402

occ = synth.config2_grid(1)
bits = torch.from_numpy(FroxelGrid.from_dense(occ).bits).cuda()
plan = PvsUNet(seed=1).plan(1, occ.shape)
plan.tune(bits)
out = torch.empty(occ.size // 8, dtype=torch.uint8, device="cuda")
plan.run(bits, out, 0.5)
torch.cuda.synchronize()
flush = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")


def timed(stop, abl):
    os.environ["FPVS_LV_STOP"], os.environ["FPVS_K2_ABL"] = stop, str(abl)
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), no_gc():
        with torch.cuda.graph(g, stream=s):
            plan.build_maps(bits, gather=True)
    torch.cuda.synchronize()
    ts = []
    for _ in range(30):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts))


k1 = timed("1", 0)
for abl in [int(v) for v in os.environ.get("ABLS", "0,1,2,4,8,16,6,31").split(",")]:
    print(f"K2_ABL {abl:3d}: K1 {k1:.1f} us, K2 (+K3 reset) {timed('2', abl) - k1:.1f} us")
os.environ["FPVS_LV_STOP"], os.environ["FPVS_K2_ABL"] = "0", "0"
