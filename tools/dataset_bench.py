"""Time the device dataset loop (dataset.PairProducer: ortho geometry + GT PVS
with the geometry OR) per frame, at the reference CLI's gen-dataset defaults
(32^3, supersample 4, 128 viewpoints -> 128^2 depth buffers) and at 256^3.

    python tools/dataset_bench.py [--frames 20] [--cpu]

--cpu also times the numpy oracle (froxelize_ortho + gt_pvs) on the first
frame at 32^3, the CPU restatement of scenegen.py:414-418.
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
    ap.add_argument("--frames", type=int, default=20)
    ap.add_argument("--cpu", action="store_true")
    a = ap.parse_args()
    import torch
    from types import SimpleNamespace
    from paper_2509_24677_b200 import synth, views
    from paper_2509_24677_b200.dataset import PairProducer
    from paper_2509_24677_b200.froxelize import FroxelizeConfig
    from paper_2509_24677_b200.gtpvs import OracleConfig
    frames = []
    for i in range(a.frames):
        v, t, fa = synth.froxel_scene(i, 12, 12)
        cell = views.ViewCell.from_forward(tuple(fa[0] + fa[5] * fa[1]), 0.3, 60.0, 15.0, tuple(fa[1]), 0.3, 20.0)
        frames.append((SimpleNamespace(vertices=v, triangles=t), cell))
    for dims in ((32, 32, 32), (256, 256, 256)):
        prod = PairProducer(dims, OracleConfig(viewpoints=128), FroxelizeConfig(supersample=4, mode="ortho"))
        prod.pair(*frames[0])
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for sc, cell in frames:
            geo, gt, ok = prod.pair(sc, cell)
        e1.record()
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) / len(frames)
        print(f"dims {dims[0]}^3: {wall * 1e3:8.2f} ms/frame wall (host setup + device), "
              f"{e0.elapsed_time(e1) / len(frames):8.2f} ms/frame between events, "
              f"{1.0 / wall:8.1f} frames/s; geometry {int(np.unpackbits(geo.cpu().numpy()).sum())} "
              f"gt {int(np.unpackbits(gt.cpu().numpy()).sum())} subset {bool(ok)}", flush=True)
    if a.cpu:
        from oracle import froxelize as ofz, gtpvs as ogt
        sc, cell = frames[0]
        fr = views.build_viewcell_frustum(cell)
        cams = views.sample_viewpoints(cell, 128)
        t0 = time.perf_counter()
        geo = ofz.froxelize_ortho(sc.vertices, sc.triangles, fr._o, fr._basis, fr.half_extent, fr.near, fr.far,
                                  (32, 32, 32), 4)
        ogt.gt_pvs(sc.vertices, sc.triangles, [c.params() for c in cams],
                   (fr._o, fr._basis, fr.half_extent, fr.near, fr.far), (32, 32, 32), (128, 128), geometry=geo)
        print(f"oracle (numpy, CPU) 32^3 frame: {time.perf_counter() - t0:.2f} s", flush=True)


if __name__ == "__main__":
    main()
