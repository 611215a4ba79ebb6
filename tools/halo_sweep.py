"""Per-layer device times of the config-2 frame: plain gather-GEMM vs the
halo-cached kernel at several (bn, split) settings (profiling aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2509_24677_b200 import synth  # noqa: E402
from paper_2509_24677_b200.froxel import FroxelGrid  # noqa: E402
from paper_2509_24677_b200.pipeline import device_stage_times  # noqa: E402
from paper_2509_24677_b200.unet import PvsUNet  # noqa: E402

occ = synth.config2_grid(1)
bits = torch.from_numpy(FroxelGrid.from_dense(occ).bits).cuda()
net = PvsUNet(seed=1, precision="bf16")
out = torch.empty(occ.size // 8, dtype=torch.uint8, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

L0 = ("enc0a", "enc0b", "dec0a", "dec0b")
L1 = ("enc1a", "enc1b", "dec1a", "dec1b")
L2 = ("enc2a", "enc2b")


def run(tag, plan):
    plan.run(bits, out, 0.5)
    torch.cuda.synchronize()
    t = device_stage_times(plan, bits, out, flush=flush)
    fl = plan.layer_flops()
    tot = sum(t.values())
    print(f"{tag:28s} total {tot * 1000:7.1f} us |",
          " ".join(f"{k}={t[k] * 1000:.1f}" for k in t), flush=True)
    print(" " * 30 + "TF/s " + " ".join(f"{k}={fl[k] / (t[k] * 1e-3) / 1e12:.0f}" for k in fl if k in t), flush=True)
    return t


plain = net.plan(1, occ.shape)
plain.use_halo, plain.halo_cfg = False, {}
plain.tune(bits)
run("plain", plain)

plan = net.plan(1, occ.shape)
plan.tune(bits)
print("auto cfg", plan.halo_cfg)
run("halo auto", plan)

from paper_2509_24677_b200 import sparse as sp  # noqa: E402
hb = sp.HaloBuilder([plan.L0, plan.L1, plan.L2])
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    hb.run()
    with torch.cuda.graph(g, stream=s):
        for _ in range(20):
            hb.run()
torch.cuda.current_stream().wait_stream(s)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
g.replay()
e1.record()
torch.cuda.synchronize()
print(f"halo build, 3 levels one launch: {e0.elapsed_time(e1) / 20 * 1000:.1f} us (device)")

rows = {k: lv.count() for k, lv in plan.level_of.items()}
variants = {
    "L2 bn256 s2": {k: (256, 2) for k in L2},
    "L2 bn256 s3": {k: (256, 3) for k in L2},
    "L2 bn256 s4": {k: (256, 4) for k in L2},
    "L2 bn128 s3": {k: (128, 3) for k in L2},
    "L1 bn128 s2": {k: (128, 2) for k in L1},
    "L0 s1": {k: (64, 1) for k in L0},
}
for tag, cfg in (variants.items() if os.environ.get("SWEEP", "1") == "1" else []):
    plan.set_halo(rows, cfg)
    run(tag, plan)
