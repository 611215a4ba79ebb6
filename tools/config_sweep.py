"""BASELINE configs 1, 3 and 4 on one B200: per-stage device times and rates.

    python tools/config_sweep.py > profiles/r1_configs.md

Config 1: the 64x64x32 tiny grid through the config-1 net (fp32 and bf16).
Config 3: the 64-grid batch (seeds 100+i, 1-6 % density) as ONE batched
frame (B = 64), grids/s.
Config 4: the config-1 net on 256^3 grids at 0.5 / 2 / 8 / 25 % occupancy:
per-stage device time (maps, sparse interleave, 4 convs, head), HBM GB/s of
the integer stages and TFLOP/s of the convs.  Each stage is captured alone
as a CUDA graph of 20 launches (pipeline.device_stage_times), L2 flushed.

Algorithmic bytes (the HBM roofline numerator):
  maps    = N/8 (packed grid read) + 7 B per cell (flag write + read, index
            volume write) + 124 B per active cell (coords 16 + neighbours 108);
  gather  = N/8 + active * d^3 * sizeof(dtype);
  convs   = useful FLOPs 2 * present pairs * Cin * Cout;
  head    = 2 * active * Cin * d^3 FLOPs (+ N/8 bytes of output).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2509_24677_b200 import synth
    from paper_2509_24677_b200.froxel import FroxelGrid
    from paper_2509_24677_b200.neural import ModelConfig, PvsNet
    from paper_2509_24677_b200.pipeline import ChainPlan, FramePipeline, device_stage_times
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                        "MEASURED_PEAKS.json"))) if os.path.exists("MEASURED_PEAKS.json") else {}
    print("# BASELINE configs 1, 3, 4 on one B200 (r1)\n")
    print("Device times from CUDA graphs of 20 launches per stage, L2 flushed "
          "(`tools/config_sweep.py`).  Peaks: " + json.dumps(peaks)[:200] + "\n")

    def frame_ms(pipe, reps=20):
        ts = []
        for _ in range(reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            pipe.run_device()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return sorted(ts)[len(ts) // 2]

    # ---- config 1
    occ1 = synth.config1_grid(0)
    print("## Config 1 (64x64x32, 200 boxes, config-1 net)\n")
    print("| precision | frame us (graph) | grids/s |")
    print("|---|---|---|")
    for prec in ("fp32", "bf16"):
        net = PvsNet(ModelConfig.config1(), np.random.Generator(np.random.PCG64(0)), precision=prec)
        pipe = FramePipeline(net, 1, occ1.shape, graph=True)
        pipe.load(torch.from_numpy(FroxelGrid.from_dense(occ1).bits).cuda())
        pipe.capture()
        ms = frame_ms(pipe)
        print(f"| {prec} | {ms * 1e3:.1f} | {1e3 / ms:.0f} |")

    # ---- config 3
    grids = [synth.config3_grid(i) for i in range(64)]
    bits = torch.from_numpy(np.concatenate([FroxelGrid.from_dense(g).bits for g in grids])).cuda()
    print("\n## Config 3 (64 grids of 64x64x32 as one batched frame, config-1 net)\n")
    print("| precision | batch frame us | grids/s (1 GPU) |")
    print("|---|---|---|")
    for prec in ("fp32", "bf16"):
        net = PvsNet(ModelConfig.config1(), np.random.Generator(np.random.PCG64(0)), precision=prec)
        pipe = FramePipeline(net, 64, (64, 64, 32), graph=True)
        pipe.load(bits)
        pipe.capture()
        ms = frame_ms(pipe)
        print(f"| {prec} | {ms * 1e3:.1f} | {64e3 / ms:.0f} |")

    # ---- config 4
    print("\n## Config 4 (config-1 net on 256^3, density sweep, bf16)\n")
    print("maps = the fused level build (flags, compaction, neighbour tables, tile masks, level-0 features, "
          "output clear: three launches); gather = n/a when fused.\n")
    print("| density | active cells | maps us | maps GB/s | gather us | gather GB/s | conv0-3 us | conv TFLOP/s "
          "| head us | frame us (graph) |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    net = PvsNet(ModelConfig.config1(), np.random.Generator(np.random.PCG64(0)), precision="bf16")
    for dens in (0.005, 0.02, 0.08, 0.25):
        occ = synth.config4_grid(dens)
        b = torch.from_numpy(FroxelGrid.from_dense(occ).bits).cuda()
        pipe = FramePipeline(net, 1, occ.shape, graph=True)
        pipe.load(b)
        pipe.capture()
        plan: ChainPlan = pipe.plan
        t = device_stage_times(plan, pipe.in_bits, pipe.out_bits, 0.5, reps=20, flush=flush)
        n = plan.L0.count()
        cells = plan.L0.ncells
        nbytes = occ.size // 8
        maps_b = nbytes + 7 * cells + 124 * n
        gath_b = nbytes + n * 8 * 2
        if "gather" not in t:  # fused level build: maps include the sparse interleave and the output clear
            maps_b += n * 8 * 2 + nbytes
            t["gather"] = float("nan")
        fl = plan.layer_flops()
        conv_ms = sum(t[k] for k in t if k.startswith("conv"))
        conv_fl = sum(fl[k] for k in fl if k.startswith("conv"))
        ms = frame_ms(pipe)
        print(f"| {occ.mean() * 100:.2f} % | {n} | {t['maps'] * 1e3:.1f} | {maps_b / (t['maps'] * 1e-3) / 1e9:.0f} | "
              f"{t['gather'] * 1e3:.1f} | {gath_b / (t['gather'] * 1e-3) / 1e9:.0f} | {conv_ms * 1e3:.1f} | "
              f"{conv_fl / (conv_ms * 1e-3) / 1e12:.0f} | {t['head'] * 1e3:.1f} | {ms * 1e3:.1f} |")
        del pipe


if __name__ == "__main__":
    main()
