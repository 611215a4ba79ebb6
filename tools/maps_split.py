"""In-frame time of the three map kernels (profiling build): graphs of
K1 / K1+K2 / K1+K2+K3 (FPVS_LV_STOP) after an L2 flush, prefix-differenced."""
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
res = {}
for stop in ("1", "2", "0"):
    os.environ["FPVS_LV_STOP"] = stop
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
    res[stop] = float(np.median(ts))
os.environ["FPVS_LV_STOP"] = "0"
print(f"K1 {res['1']:.1f} us | K2 {res['2'] - res['1']:.1f} | K3 {res['0'] - res['2']:.1f} | maps {res['0']:.1f}")
