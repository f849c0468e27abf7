"""Build the in-tree CUDA library (sm_100a) behind the C ABI.

    python -m paper_2003_08646_b200.build

Produces paper_2003_08646_b200/_build/liblance_b200.so with nvcc directly (no
torch types anywhere in the library).  -fmad=false and no fast-math: the
path is bit-exact with the reference only without FMA contraction
(SURVEY.md Appendix A).
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT_DIR = os.path.join(PKG, "_build")
LIB = os.path.join(OUT_DIR, "liblance_b200.so")
SOURCES = ["lance_input.cu", "lance_filter.cu", "lance_gemm.cu", "lance_f4.cu", "lance_stack.cu", "lance_abi.cu"]
HEADERS = ["lance_common.cuh", "lance_kernels.cuh", "lance_ptx.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-DLANCE_JMAJOR=" + os.environ.get("LANCE_JMAJOR", "0"), "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-fmad=false",
         "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "-I" + os.path.join(ROOT, "include")]
# LANCE_PROFILING=1: honour the experiment / A-B environment switches
# (lance_knob) -- tools/*.sh only; release builds ignore the environment.
if os.environ.get("LANCE_PROFILING"):
    FLAGS.append("-DLANCE_PROFILING")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "lance_b200.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    os.makedirs(OUT_DIR, exist_ok=True)
    objs = [os.path.join(OUT_DIR, src.replace(".cu", ".o")) for src in SOURCES]

    def compile_one(src_obj):
        src, obj = src_obj
        cmd = [NVCC, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        list(ex.map(compile_one, zip(SOURCES, objs)))
    tmp = LIB + ".tmp"
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs]
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
