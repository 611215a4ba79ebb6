"""A/B builds of the product library: recompile one or more csrc files with
extra -D flags and link against the rest of the product objects into
paper_2509_24677_b200/libfpvs_<name>.so (git-ignored; travels with gpurun).
Load it with FPVS_LIB=... (e.g. tools/frame_variant.py in two processes).

  python tools/build_variant.py NAME FILE.cu[,FILE2.cu] -DMACRO=VALUE ...
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_24677_b200 import build as B  # noqa: E402

name, files, defines = sys.argv[1], sys.argv[2].split(","), sys.argv[3:]
B.build(verbose=False)
objdir = os.path.join(B.HERE, "_build")
vdir = os.path.join(B.HERE, "_build_" + name)
os.makedirs(vdir, exist_ok=True)
objs = []
for src in B.SOURCES:
    if src in files:
        obj = os.path.join(vdir, src.replace(".cu", ".o"))
        subprocess.check_call([B.nvcc(), *B.ARCH, *B.FLAGS, *defines, "-c", os.path.join(B.CSRC, src), "-o", obj])
    else:
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
    objs.append(obj)
out = os.path.join(B.HERE, f"libfpvs_{name}.so")
subprocess.check_call([B.nvcc(), *B.ARCH, "-shared", "-o", out, *objs])
print(out)
