"""Per-role timestamps of the halo conv for CTA 0 (FPVS_HALO_DEBUG=1)."""
import ctypes
import os
import sys

os.environ["FPVS_HALO_DEBUG"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
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
plan.run(bits, out, 0.5)
stages = dict(plan.stages(bits, out, 0.5))
lib = _lib.load()
buf = (ctypes.c_ulonglong * (2 * 8192))()
for name in os.environ.get("LAYERS", "enc0b,enc1a,enc2a").split(","):
    for _ in range(3):
        torch.cuda.synchronize()
        ctypes.memset(buf, 0, ctypes.sizeof(buf))
        stages[name]()
        torch.cuda.synchronize()
    lib.fpvs_debug_halo_timestamps(buf, 2 * 8192)
    t = np.frombuffer(buf, dtype=np.uint64)[:8192].astype(np.int64)
    t0 = t[0]
    rel = lambda v: (v - t0) / 1000.0 if v else float("nan")  # noqa: E731
    print(f"=== {name} cfg {plan.halo_cfg.get(name)}  start->setup {rel(t[1]):.2f}  main end {rel(t[2]):.2f}  "
          f"exit {rel(t[3]):.2f} us")
    for g in range(8):
        if not t[16 + 3 * g]:
            break
        print(f"  group {g}: loader hempty {rel(t[16 + 3 * g]):7.2f} meta {rel(t[17 + 3 * g]):7.2f} "
              f"issued {rel(t[18 + 3 * g]):7.2f} | builders ready g0 {rel(t[256 + 4 * g]):7.2f} "
              f"g1 {rel(t[258 + 4 * g]):7.2f} done g0 {rel(t[257 + 4 * g]):7.2f} g1 {rel(t[259 + 4 * g]):7.2f}")
    for it in range(8):
        if not t[7000 + 2 * it]:
            break
        print(f"  unit {it}: mma tempty {rel(t[7000 + 2 * it]):7.2f} tfull {rel(t[7001 + 2 * it]):7.2f} "
              f"epi got {rel(t[7200 + 2 * it]):7.2f}")
    kc = 0
    rows = []
    while t[4096 + 2 * kc] and kc < 1000:
        rows.append((rel(t[1024 + 3 * kc]), rel(t[1025 + 3 * kc]), rel(t[1026 + 3 * kc]), rel(t[4096 + 2 * kc]),
                     rel(t[4097 + 2 * kc])))
        kc += 1
    r = np.array(rows)
    print(f"  chunks {kc}: mma full-wait-done interval mean {np.nanmean(np.diff(r[:, 3])):.3f} us; "
          f"builder lds->arrive mean {np.nanmean(r[:, 2] - r[:, 0]):.3f}; empty wait mean "
          f"{np.nanmean(r[:, 1] - r[:, 0]):.3f}; arrive->mma mean {np.nanmean(r[:, 3] - r[:, 2]):.3f}")
    for i in list(range(0, min(kc, 12))) + list(range(26, min(kc, 34))):
        print("   kc %3d  lds %7.2f empty %7.2f arrive %7.2f | mma full %7.2f commit %7.2f" % ((i,) + rows[i]))
