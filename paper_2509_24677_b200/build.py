"""Build libfpvs.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

The library is a plain C-ABI shared object (include/fpvs.h) so that any
host language can bind it; the Python package loads it with ctypes.  It is
written next to this file so it travels to the GPU box with the repo
snapshot.  Usage: ``python -m paper_2509_24677_b200.build``.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libfpvs.so")
PROFILE_LIB = os.path.join(HERE, "libfpvs_prof.so")  # -DFPVS_PROFILE: timestamps + ablation knobs (tools/ only)
SOURCES = ["capi.cu", "interleave.cu", "kmap.cu", "kmap_pairs.cu", "levels.cu", "spconv_simt.cu", "spconv_tc.cu", "spconv_halo.cu", "spconv_brick.cu", "upsort.cu", "wgrad_tc.cu", "wgrad_halo.cu", "optim.cu", "froxelize.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr",
         "-diag-suppress", "177"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(lib) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(HERE, "..", "include", "fpvs.h")]
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def build(force: bool = False, verbose: bool = True, profile: bool = False) -> str:
    """Compile every .cu under csrc/ into libfpvs.so (parallel per-file objects).

    ``profile`` builds libfpvs_prof.so instead, with -DFPVS_PROFILE: per-role
    timestamp buffers, the FPVS_*_DEBUG / FPVS_HALO_ABL knobs and the
    fpvs_debug_* read-out entry points (tools/halo_timeline.py, halo_ablate.py
    load it through FPVS_LIB).  The product library never contains them."""
    lib = PROFILE_LIB if profile else LIB
    if not force and not _stale(lib):
        return lib
    objdir = os.path.join(HERE, "_build_prof" if profile else "_build")
    os.makedirs(objdir, exist_ok=True)
    cc = nvcc()
    procs = []
    objs = []
    for src in SOURCES:
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        objs.append(obj)
        cmd = [cc, *ARCH, *FLAGS, *(["-DFPVS_PROFILE"] if profile else []), "-c", os.path.join(CSRC, src), "-o", obj]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    for src, p in procs:
        out = p.communicate()[0].decode()
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{out}")
        if verbose and out.strip():
            print(out, file=sys.stderr)
    tmp = lib + ".tmp"
    subprocess.check_call([cc, *ARCH, "-shared", "-o", tmp, *objs])
    os.replace(tmp, lib)
    if verbose:
        print(f"built {lib}", file=sys.stderr)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, profile="--profile" in sys.argv)
