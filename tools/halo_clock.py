"""Cycle-level per-stage timing of one halo conv CTA (profiling build, clock64):
MMA full-wait / issue / commit and builder empty-wait / work per stage.

LAYERS=enc0b ABL=<FPVS_HALO_ABL bits>"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("FPVS_LIB", os.path.join(ROOT, "paper_2509_24677_b200", "libfpvs_prof.so"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_24677_b200 import _lib, synth  # noqa: E402
from paper_2509_24677_b200.froxel import FroxelGrid  # noqa: E402
from paper_2509_24677_b200.unet import PvsUNet  # noqa: E402

occ = synth.config2_grid(1)
bits = torch.from_numpy(FroxelGrid.from_dense(occ).bits).cuda()
plan = PvsUNet(seed=1).plan(1, occ.shape)
plan.tune(bits)
out = torch.empty(occ.size // 8, dtype=torch.uint8, device="cuda")
plan.overlap = False
plan.run(bits, out, 0.5)
stages = dict(plan.stages(bits, out, 0.5))
lib = _lib.load()
buf = (ctypes.c_ulonglong * (2 * 8192))()
cta = int(os.environ.get("CTA", "40"))
import itertools  # noqa: E402
abls = [int(v) for v in os.environ.get("ABLS", os.environ.get("ABL", "0")).split(",")]
for name, abl in itertools.product(os.environ.get("LAYERS", "enc0b,enc1a").split(","), abls):
    os.environ["FPVS_HALO_ABL"] = str(abl)
    os.environ["FPVS_HALO_DEBUG"] = str(1 + 128 + 256 * cta)
    for _ in range(3):
        torch.cuda.synchronize()
        ctypes.memset(buf, 0, ctypes.sizeof(buf))
        stages[name]()
        torch.cuda.synchronize()
    os.environ["FPVS_HALO_DEBUG"] = "0"
    lib.fpvs_debug_halo_timestamps(buf, 2 * 8192)
    t = np.frombuffer(buf, dtype=np.uint64)[:8192].astype(np.int64)
    n = 0
    while n < 400 and t[4096 + 2 * n] and t[3600 + n]:
        n += 1
    st = np.arange(n)
    mwait0, mstart, mcommit = t[3600 + st], t[4096 + 2 * st], t[4097 + 2 * st]
    os.environ["FPVS_HALO_ABL"] = "0"
    print(f"=== {name} abl {abl:#x}: CTA {cta}, {n} stages, total {t[2] - t[1]} cycles (main loop), cfg {plan.halo_cfg.get(name)}")
    print(f"  MMA thread per stage: full-wait {np.median(mstart - mwait0):.0f} cyc (mean {np.mean(mstart - mwait0):.0f}), "
          f"issue {np.median(mcommit - mstart):.0f} (mean {np.mean(mcommit - mstart):.0f}), "
          f"stage period {np.median(np.diff(mstart)):.0f} (mean {np.mean(np.diff(mstart)):.0f})")
    for bg in (0, 1):
        pre, post, arr = t[2000 + 2 * st + bg], t[2800 + 2 * st + bg], t[1024 + 2 * st + bg]
        lds0 = t[5400 + 2 * st + bg]
        ok = (pre > 0) & (post > 0) & (arr > 0) & (lds0 > 0)
        if ok.any():
            print(f"  builder group {bg}: halo reads {np.median((pre - lds0)[ok]):.0f} (mean {np.mean((pre - lds0)[ok]):.0f}), "
                  f"prev arrive -> reads {np.median((lds0[1:] - arr[:-1])[ok[1:] & ok[:-1]]):.0f}, "
                  f"empty-wait {np.median((post - pre)[ok]):.0f} (mean {np.mean((post - pre)[ok]):.0f}), "
                  f"wait-end -> arrive {np.median((arr - post)[ok]):.0f}, arrive -> MMA start {np.median((mstart - arr)[ok]):.0f}")
    if os.environ.get("BRIEF"):
        continue
    print("  first stages (cycles from MMA start of stage 0):")
    base = mstart[0]
    for i in range(min(n, 12)):
        print(f"   st {i:3d}: mma wait {mwait0[i] - base:7d} start {mstart[i] - base:7d} commit {mcommit[i] - base:7d} | "
              f"b0 pre {t[2000 + 2 * i] - base:7d} post {t[2800 + 2 * i] - base:7d} arr {t[1024 + 2 * i] - base:7d} | "
              f"b1 pre {t[2001 + 2 * i] - base:7d} post {t[2801 + 2 * i] - base:7d} arr {t[1025 + 2 * i] - base:7d}")
    # per-halo (tile) events: loader hempty-wait end / meta landed / copies issued, builders' halo ready
    print("  halo buffers (cycles from MMA start of stage 0):")
    for gc in range(4):
        ev = [t[16 + 3 * gc], t[17 + 3 * gc], t[18 + 3 * gc], t[256 + 4 * gc], t[258 + 4 * gc], t[257 + 4 * gc]]
        if not ev[0]:
            break
        print(f"   halo {gc}: loader free {ev[0] - base:7d} meta {ev[1] - base:7d} issued {ev[2] - base:7d} | "
              f"b0 at hfull-wait {ev[5] - base if ev[5] else 0:7d} ready {ev[3] - base:7d} b1 ready {ev[4] - base if ev[4] else 0:7d}")
    print("  builder b0 per halo: " + " ".join(f"[top {t[6000 + 4 * g] - base} meta-ok {t[6001 + 4 * g] - base} "
                                              f"loop-end {t[6002 + 4 * g] - base} hempty-arrived {t[6003 + 4 * g] - base} | next unit top {t[7802 + 2 * g] - base} "
                                              f"got unit {t[7803 + 2 * g] - base}]" for g in range(3) if t[6000 + 4 * g]))
    print("  unit boundaries (MMA): " + " ".join(f"u{k}: acc-wait {t[7601 + 2 * k] - base} -> {t[7000 + 2 * k] - base}, "
                                                    f"done {t[7001 + 2 * k] - base}" for k in range(3) if t[7000 + 2 * k]))
    print("  epilogue tile start: " + " ".join(str(t[7200 + 2 * k] - base) for k in range(3) if t[7200 + 2 * k]))
