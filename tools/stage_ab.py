"""Per-stage in-frame device times (pipeline.frame_stage_times: L2-flushed
prefix graphs) of the config-2 frame for a few environment variants, side
by side.  VARIANTS as tools/frame_variant.py (';' between variants, ','
between ENV=VAL)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2509_24677_b200 import synth  # noqa: E402
from paper_2509_24677_b200.froxel import FroxelGrid  # noqa: E402
from paper_2509_24677_b200.pipeline import FramePipeline, frame_stage_times  # noqa: E402
from paper_2509_24677_b200.unet import PvsUNet  # noqa: E402

variants = os.environ.get("VARIANTS", "FPVS_BRICK=;FPVS_BRICK=2").split(";")
occ = synth.config2_grid(1)
bits = torch.from_numpy(FroxelGrid.from_dense(occ).bits).cuda()
flush = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
res = []
for var in variants:
    saved = {}
    for kv in var.split(","):
        if "=" in kv:
            k, v = kv.split("=", 1)
            saved[k] = os.environ.get(k)
            os.environ[k] = v
    pipe = FramePipeline(PvsUNet(seed=1), 1, occ.shape)
    pipe.load(bits)
    pipe.capture()
    st, frame = frame_stage_times(pipe.plan, pipe.in_bits, pipe.out_bits, 0.5, flush=flush, reps=int(os.environ.get("REPS", "20")))
    res.append((var, st, frame))
    for k, v in saved.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v
    del pipe
names = list(res[0][1])
print("stage    " + "  ".join(f"{v[:18]:>18s}" for v, _, _ in res))
for n in names:
    print(f"{n:8s} " + "  ".join(f"{st.get(n, 0) * 1e3:18.2f}" for _, st, _ in res))
print("frame    " + "  ".join(f"{f * 1e3:18.2f}" for _, _, f in res))
