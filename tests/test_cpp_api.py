"""The C++ host API (include/lance/b200.hpp) as a reference-style C++ caller
uses it: examples/cpp_drop_in.cpp is compiled with g++ against the in-tree
library.  CPU: it builds and fails loudly without a device (no CPU fallback).
GPU: its checksum line equals the oracle's output (F(2x2) and F(4x4))."""
import os
import shutil
import subprocess

import pytest

from oracle import Oracle, Spec
from paper_2003_08646_b200 import _lib, tensor_io

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build_example(tmp_path):
    if shutil.which("g++") is None:
        pytest.skip("g++ not available")
    _lib.lib()  # builds the library when stale
    libdir = os.path.join(ROOT, "paper_2003_08646_b200", "_build")
    exe = str(tmp_path / "cpp_drop_in")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "cpp_drop_in.cpp"), "-L" + libdir,
                    "-llance_b200", "-Wl,-rpath," + libdir, "-o", exe], check=True)
    return exe


def test_cpp_example_builds_and_has_no_cpu_fallback(tmp_path):
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("device present")
    exe = build_example(tmp_path)
    r = subprocess.run([exe, "1", "8", "8", "8", "4", "1", "42", "2"], capture_output=True, text=True)
    assert r.returncode == 1 and "no CPU fallback" in r.stderr
    r = subprocess.run([exe, "1", "8", "8", "8", "4", "2", "42", "2"], capture_output=True, text=True)
    assert r.returncode == 2 and "pad must be 0 or 1" in r.stderr  # validation before any device work


@pytest.mark.gpu
@pytest.mark.parametrize("tile_m", [2, 4])
def test_cpp_example_matches_oracle(tmp_path, tile_m):
    exe = build_example(tmp_path)
    spec = Spec(2, 16, 10, 10, 8, 1)
    r = subprocess.run([exe, "2", "16", "10", "10", "8", "1", "42", str(tile_m)],
                       capture_output=True, text=True, check=True)
    o = Oracle()
    x, w = o.layer(spec, 42)
    y = o.lance_gemm(spec, x, w, tile_m=tile_m)
    assert r.stdout.strip() == f"output dims 2 10 10 8  checksum {tensor_io.fnv1a64(y):x}"
