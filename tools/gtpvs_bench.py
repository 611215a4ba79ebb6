"""Time fpvs_gt_pvs (device) on synthetic scenes; optional oracle timing on a few cameras.

    python tools/gtpvs_bench.py [--dims 256] [--views 128] [--cpu-views 2]
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
    ap.add_argument("--views", type=int, default=128)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--cpu-views", type=int, default=0)
    ap.add_argument("--scenes", default="0,1")
    a = ap.parse_args()
    import torch
    from paper_2509_24677_b200 import gtpvs, synth, views
    from oracle import gtpvs as ogt
    dims = (a.dims,) * 3
    scenes = [(0, 12, 12), (1, 40, 24), (2, 200, 48)]
    for si in a.scenes.split(","):
        seed, nobj, detail = scenes[int(si)]
        v, t, fa = synth.froxel_scene(seed, nobj, detail)
        origin, fwd = fa[0], fa[1]
        cell = views.ViewCell.from_forward(tuple(origin + fa[5] * fwd), 0.3, 60.0, 15.0, tuple(fwd), 0.3, 20.0)
        ocfg = gtpvs.OracleConfig(viewpoints=a.views)
        g = gtpvs.GtPvs(v, t)
        out = g.for_cell(cell, dims, ocfg)
        torch.cuda.synchronize()
        samples = g.samples() if hasattr(g, "samples") else -1
        best = 1e9
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.for_cell(cell, dims, ocfg, out=None)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        got = out.cpu().numpy()
        line = (f"scene{seed} tris {len(t):7d} views {a.views} res {ocfg.resolution_for(dims)} "
                f"gt {int(np.unpackbits(got).sum()):8d}  {best:8.2f} ms ({best / a.views * 1e3:7.1f} us/view)")
        if a.cpu_views:
            cams = views.sample_viewpoints(cell, a.views)[:a.cpu_views]
            fr = views.build_viewcell_frustum(cell)
            t0 = time.perf_counter()
            ogt.gt_pvs(v, t, [c.params() for c in cams], (fr._o, fr._basis, fr.half_extent, fr.near, fr.far), dims,
                       ocfg.resolution_for(dims))
            dt = time.perf_counter() - t0
            line += f"  oracle {dt / a.cpu_views:.2f} s/view"
        print(line, flush=True)


if __name__ == "__main__":
    main()
