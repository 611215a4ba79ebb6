"""Frame device time (CUDA graph replay, L2 flushed) under plan variants: A/B aid."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2509_24677_b200 import synth  # noqa: E402
from paper_2509_24677_b200.froxel import FroxelGrid  # noqa: E402
from paper_2509_24677_b200.pipeline import FramePipeline  # noqa: E402
from paper_2509_24677_b200.unet import PvsUNet  # noqa: E402


def frame_ms(pipe, reps=30):
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pipe.run_device()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


occ = synth.config2_grid(1)
bits = torch.from_numpy(FroxelGrid.from_dense(occ).bits).cuda()
for variant in os.environ.get("VARIANTS", "default,no_overlap").split(","):
    net = PvsUNet(seed=1, precision="bf16")
    pipe = FramePipeline(net, 1, occ.shape, tau=0.5, graph=True)
    pipe.load(bits)
    if variant == "no_overlap":
        pipe.plan.overlap = False
    pipe.capture()
    print(f"{variant:12s} PDL={os.environ.get('FPVS_PDL', '1')}  frame {frame_ms(pipe) * 1000:.1f} us", flush=True)
