"""Per-role timestamps of the halo conv for CTA 0 (FPVS_HALO_DEBUG=1).

LAYERS=enc0b,enc1a,enc2a  HALO_CFG="64,1;128,1;256,1" (bn,split per level)."""
import ctypes
import os
import sys

os.environ.setdefault("FPVS_HALO_DEBUG", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
# timestamps / ablations exist only in the profiling build (python -m paper_2509_24677_b200.build --profile)
os.environ.setdefault("FPVS_LIB", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                               "paper_2509_24677_b200", "libfpvs_prof.so"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_24677_b200 import _lib, synth  # noqa: E402
from paper_2509_24677_b200.froxel import FroxelGrid  # noqa: E402
from paper_2509_24677_b200.unet import PvsUNet  # noqa: E402

occ = synth.config2_grid(1)
bits = torch.from_numpy(FroxelGrid.from_dense(occ).bits).cuda()
plan = PvsUNet(seed=1).plan(1, occ.shape)
plan.tune(bits)
cfg = os.environ.get("HALO_CFG")
if cfg:
    per = [tuple(int(v) for v in c.split(",")) for c in cfg.split(";")]
    rows = {k: lv.count() for k, lv in plan.level_of.items()}
    plan.set_halo(rows, {k: per[int(k[-2])] for k in rows})
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
    cta = (ctypes.c_ulonglong * (32 * 3 * 160))()
    if hasattr(lib, "fpvs_debug_halo_cta_times"):
        lib.fpvs_debug_halo_cta_times(cta)
    spans = np.frombuffer(cta, dtype=np.uint64).astype(np.int64).reshape(32, 3, 160)
    ca = spans[int(np.argmax(spans[:, 0].max(axis=1)))]  # the latest launch's slot
    ok = (ca[0] > 0) & (ca[1] > ca[0])
    st_, en_ = ca[0][ok], ca[1][ok]
    if len(st_):
        t00 = st_.min()
        d = (en_ - st_) / 1000.0
        print(f"  CTAs {ok.sum()}: launch span {(en_.max() - t00) / 1000:.2f} us; start spread {(st_.max() - t00) / 1000:.2f} us; "
              f"CTA duration min {d.min():.2f} median {np.median(d):.2f} max {d.max():.2f} us")
        idx = np.nonzero(ok)[0]
        if hasattr(lib, "fpvs_debug_halo_clk"):
            ck = (ctypes.c_longlong * 320)()
            lib.fpvs_debug_halo_clk(ck)
            ck = np.frombuffer(ck, dtype=np.int64).reshape(2, 160)
            f = (ck[1][ok] - ck[0][ok]) / np.maximum(en_ - st_, 1)
            print(f"   SM clock over the CTA: median {np.median(f) * 1e3:.0f} MHz (min {f.min() * 1e3:.0f}, max {f.max() * 1e3:.0f})")
        print("   durations by CTA:", " ".join(f"{i}:{x:.1f}" for i, x in zip(idx[:40], d[:40])))
        sm = (ctypes.c_uint * 160)()
        if hasattr(lib, "fpvs_debug_halo_smid"):
            lib.fpvs_debug_halo_smid(sm)
            print("   smid:", " ".join(str(v) for v in list(sm)[:40]))
    t = np.frombuffer(buf, dtype=np.uint64)[:8192].astype(np.int64)
    t0 = t[0]
    rel = lambda v: (v - t0) / 1000.0 if v else float("nan")  # noqa: E731
    print(f"=== {name} cfg {plan.halo_cfg.get(name)}  setup {rel(t[1]):.2f}  main end {rel(t[2]):.2f}  "
          f"exit {rel(t[3]):.2f} us")
    for g in range(6):
        if not t[16 + 3 * g]:
            break
        print(f"  halo group {g}: loader hempty {rel(t[16 + 3 * g]):7.2f} meta {rel(t[17 + 3 * g]):7.2f} "
              f"issued {rel(t[18 + 3 * g]):7.2f} | builders ready g0 {rel(t[256 + 4 * g]):7.2f} g1 {rel(t[258 + 4 * g]):7.2f}")
    for it in range(6):
        if not t[7000 + 2 * it]:
            break
        print(f"  unit {it}: mma tempty {rel(t[7000 + 2 * it]):7.2f} tfull {rel(t[7001 + 2 * it]):7.2f} "
              f"epi got {rel(t[7200 + 2 * it]):7.2f} | loop top {rel(t[7600 + 2 * it]):7.2f} "
              f"unit_of done {rel(t[7601 + 2 * it]):7.2f} | split: partial written {rel(t[7400 + 4 * it]):7.2f} "
              f"counted {rel(t[7402 + 4 * it]):7.2f} "
              f"reduced {rel(t[7403 + 4 * it]):7.2f}")
    rows = []
    st = 0
    while st < 450 and t[4096 + 2 * st]:
        rows.append((rel(t[5000 + st]), rel(t[1024 + 2 * st]), rel(t[1025 + 2 * st]), rel(t[4096 + 2 * st]),
                     rel(t[4097 + 2 * st])))
        st += 1
    r = np.array(rows)
    bmax = np.fmax(r[:, 1], r[:, 2])
    print(f"  stages {st}: mma start interval {np.nanmean(np.diff(r[:, 3])):.3f} us | mma start - last builder "
          f"{np.nanmean(r[:, 3] - bmax):.3f} | mma start - B issue {np.nanmean(r[:, 3] - r[:, 0]):.3f} | "
          f"issue->commit {np.nanmean(r[:, 4] - r[:, 3]):.3f}")
    ch = []
    for i in range(min(st, 200)):
        prev = t[4096 + 2 * i]
        for g in range(4):
            v = t[6000 + 4 * i + g]
            if v and prev:
                ch.append((v - prev) / 1000.0)
                prev = v
    if ch:
        ch = np.array(ch)
        print(f"  per-chunk (4 MMA) issue time: mean {ch.mean():.3f} us, median {np.median(ch):.3f}, p10 {np.percentile(ch, 10):.3f}, p90 {np.percentile(ch, 90):.3f}")
    for i in list(range(0, min(st, 10))) + list(range(max(10, st - 4), st)):
        print("   st %3d  B issued %7.2f | built g0 %7.2f g1 %7.2f | mma start %7.2f commit %7.2f" % ((i,) + rows[i]))
    if os.environ.get("PEER"):
        t1 = np.frombuffer(buf, dtype=np.uint64)[8192:].astype(np.int64)
        rel1 = lambda v: (v - t0) / 1000.0 if v else float("nan")  # noqa: E731
        print("  peer CTA (block 1), same clock:")
        for i in range(0, 10):
            print("   st %3d  B issued %7.2f | built g0 %7.2f g1 %7.2f | full seen %7.2f forwarded %7.2f" % (
                i, rel1(t1[5000 + i]), rel1(t1[1024 + 2 * i]), rel1(t1[1025 + 2 * i]), rel1(t1[4096 + 2 * i]),
                rel1(t1[4097 + 2 * i])))
