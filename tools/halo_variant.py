"""A/B a halo-conv build variant inside the real config-2 frame (profiling build).

VAR=FPVS_HALO_NBG VALS=2,4: for each value the env knob is set, the frame's
output bits are checked against the first value's (bit-exact) and the
per-stage in-frame times (pipeline.frame_stage_times) are printed side by side.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("FPVS_LIB", os.path.join(ROOT, "paper_2509_24677_b200", "libfpvs_prof.so"))
import torch  # noqa: E402

from paper_2509_24677_b200 import synth  # noqa: E402
from paper_2509_24677_b200.froxel import FroxelGrid  # noqa: E402
from paper_2509_24677_b200.pipeline import frame_stage_times  # noqa: E402
from paper_2509_24677_b200.unet import PvsUNet  # noqa: E402

var = os.environ.get("VAR", "FPVS_HALO_NBG")
vals = os.environ.get("VALS", "2,4").split(",")
occ = synth.config2_grid(int(os.environ.get("SEED", "1")))
bits = torch.from_numpy(FroxelGrid.from_dense(occ).bits).cuda()
plan = PvsUNet(seed=1).plan(1, occ.shape)
plan.tune(bits)
flush = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
res, ref = {}, None
for v in vals:
    os.environ[var] = v
    out = torch.zeros(occ.size // 8, dtype=torch.uint8, device="cuda")
    plan.run(bits, out, 0.5)
    torch.cuda.synchronize()
    if ref is None:
        ref = out.clone()
    same = bool(torch.equal(out, ref))
    t, frame = frame_stage_times(plan, bits, out, 0.5, flush=flush, reps=int(os.environ.get("REPS", "20")))
    res[v] = (t, frame, same)
names = list(res[vals[0]][0])
print(f"{var}: " + "  ".join(f"{v:>9s}" for v in vals))
for n in names:
    print(f"{n:8s} " + "  ".join(f"{res[v][0][n] * 1e3:9.2f}" for v in vals))
print("frame    " + "  ".join(f"{res[v][1] * 1e3:9.2f}" for v in vals))
print("bitexact " + "  ".join(f"{str(res[v][2]):>9s}" for v in vals))
