"""Build A/B variants of the library that differ in one CUDA source.

    python tools/ab_build.py NAME lance_gemm.cu path/to/variant.cu [lance_abi.cu path/to/v2.cu ...]

Reuses the other objects of the current in-tree build (run the normal build
first) and writes scratch/ab_NAME/liblance_b200.so; select it at run time with
LANCE_LIB_PATH (paper_2003_08646_b200/_lib.py).  Experiments only.
"""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2003_08646_b200 import build as B  # noqa: E402

name = sys.argv[1]
pairs = [(sys.argv[i], os.path.abspath(sys.argv[i + 1])) for i in range(2, len(sys.argv), 2)]
out = os.path.join(ROOT, "scratch", "ab_" + name)
os.makedirs(out, exist_ok=True)
swapped = {}
for target, src in pairs:
    # compile the variant inside csrc so its relative includes resolve
    tmp_src = os.path.join(B.CSRC, "_ab_" + name + "_" + target)
    shutil.copy(src, tmp_src)
    try:
        obj = os.path.join(out, target.replace(".cu", ".o"))
        subprocess.run([B.NVCC, *B.FLAGS, "-c", tmp_src, "-o", obj], check=True)
    finally:
        os.remove(tmp_src)
    swapped[target] = obj
objs = [swapped.get(s, os.path.join(B.OUT_DIR, s.replace(".cu", ".o"))) for s in B.SOURCES]
subprocess.run([B.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o",
                os.path.join(out, "liblance_b200.so"), *objs], check=True)
print(os.path.join(out, "liblance_b200.so"))
