"""Throughput of back-to-back frames: one pipeline on one stream vs two
pipelines (separate buffers) alternating on two streams."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2509_24677_b200 import synth  # noqa: E402
from paper_2509_24677_b200.froxel import FroxelGrid  # noqa: E402
from paper_2509_24677_b200.pipeline import FramePipeline  # noqa: E402
from paper_2509_24677_b200.unet import PvsUNet  # noqa: E402

occ = synth.config2_grid(1)
bits = torch.from_numpy(FroxelGrid.from_dense(occ).bits).cuda()
net = PvsUNet(seed=1, precision="bf16")
pipes = []
for k in range(int(os.environ.get("NPIPES", "3"))):
    p = FramePipeline(net, 1, occ.shape, tau=0.5, graph=True)
    p.load(bits)
    p.capture()
    pipes.append(p)
streams = [torch.cuda.Stream() for _ in pipes]
N = 64
for npipe in range(1, len(pipes) + 1):
    for rep in range(2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cur = torch.cuda.current_stream()
        e0.record(cur)
        for s in streams[:npipe]:
            s.wait_stream(cur)
        for i in range(N):
            k = i % npipe
            with torch.cuda.stream(streams[k]):
                pipes[k].run_device()
        for s in streams[:npipe]:
            cur.wait_stream(s)
        e1.record(cur)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{npipe} pipeline(s): {N} frames in {ms:.2f} ms -> {ms / N * 1000:.1f} us/frame, {N / ms * 1000:.0f} grids/s",
          flush=True)
ref = pipes[0].out_bits.clone()
for p in pipes[1:]:
    assert torch.equal(p.out_bits, ref)
print("outputs identical")
