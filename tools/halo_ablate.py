"""Ablation timing of the halo conv (temporary FPVS_HALO_DEBUG bits, results are wrong
by construction): which data movement bounds a layer.

  bit 16: weight chunks loaded only for the first NS stages (B TMA traffic off)
  bit 17: builders skip the smem halo reads (zero A rows)
  bit 18: builders skip tcgen05.st
  bit 19: halo loaders skip the cp.async row copies
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
# timestamps / ablations exist only in the profiling build (python -m paper_2509_24677_b200.build --profile)
os.environ.setdefault("FPVS_LIB", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                               "paper_2509_24677_b200", "libfpvs_prof.so"))
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
plan.overlap = False
plan.run(bits, out, 0.5)
torch.cuda.synchronize()
stages = dict(plan.stages(bits, out, 0.5))
layers = os.environ.get("LAYERS", "enc0a,enc0b,enc1a,enc2a,dec1a,dec0a").split(",")
flags = {"base": 0, "noB": 1 << 16, "noLDS": 1 << 17, "noTST": 1 << 18, "noHalo": 1 << 19,
         "noLDS+noB": (1 << 16) | (1 << 17), "noLDS+noB+noHalo": (1 << 16) | (1 << 17) | (1 << 19),
         "all": (1 << 16) | (1 << 17) | (1 << 18) | (1 << 19), "noMMA": 1 << 20,
         "all+noMMA": 0x1F0000}
print("layer     " + " ".join(f"{k:>17s}" for k in flags))
for name in layers:
    row = []
    for fname, f in flags.items():
        os.environ["FPVS_HALO_ABL"] = str(f)
        fn = stages[name]
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s), no_gc():
            with torch.cuda.graph(g, stream=s):
                for _ in range(20):
                    fn()
        torch.cuda.current_stream().wait_stream(s)
        best = 1e9
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) / 20 * 1e3)
        row.append(best)
        del g
    print(f"{name:9s} " + " ".join(f"{v:17.2f}" for v in row))
os.environ["FPVS_HALO_ABL"] = "0"
