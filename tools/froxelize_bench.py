"""Time fpvs_froxelize on synthetic scenes (device time, CUDA graph of R calls).

    python tools/froxelize_bench.py [--dims 256] [--ss 4] [--mode ortho]
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", type=int, default=256)
    ap.add_argument("--ss", type=int, default=4)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--cpu", action="store_true", help="also time the oracle port")
    ap.add_argument("--scenes", default="0,1,2,3")
    ap.add_argument("--mode", default="perspective", choices=["perspective", "ortho"])
    a = ap.parse_args()
    import torch
    from paper_2509_24677_b200 import synth
    from paper_2509_24677_b200.froxelize import FroxelizeConfig, Froxelizer, Frustum
    from oracle import froxelize as ofz
    dims = (a.dims,) * 3
    cfg = FroxelizeConfig(supersample=a.ss, mode=a.mode)
    scenes = [(0, 12, 12), (1, 40, 24), (2, 200, 48), (3, 2000, 24)]
    for seed, nobj, detail in [scenes[int(i)] for i in a.scenes.split(",")]:
        v, t, fa = synth.froxel_scene(seed, nobj, detail)
        fr = Frustum.from_vectors(*fa)
        fz = Froxelizer(v, t)
        out = torch.empty(int(np.prod(dims)) // 8, dtype=torch.uint8, device="cuda")
        fz.run(fr, dims, cfg, out=out)
        torch.cuda.synchronize()
        ns = fz.samples()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                for _ in range(a.reps):
                    fz.run(fr, dims, cfg, out=out)
        torch.cuda.current_stream().wait_stream(s)
        best = 1e9
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) / a.reps)
        got = out.cpu().numpy()
        line = (f"scene{seed} tris {len(t):7d} samples {ns / 1e6:7.2f} M occupied {int(np.unpackbits(got).sum()):8d} "
                f"device {best * 1e3:8.1f} us  {ns / best / 1e6:7.2f} Gsample/s")
        if a.cpu and len(t) < 50000:
            t0 = time.perf_counter()
            fn = ofz.froxelize_ortho if a.mode == "ortho" else ofz.froxelize
            ref = fn(v, t, fr._o, fr._basis, fr.half_extent, fr.near, fr.far, dims, a.ss)
            line += f"  oracle {time.perf_counter() - t0:6.2f} s  match {np.array_equal(ref, got)}"
        print(line, flush=True)


if __name__ == "__main__":
    main()
