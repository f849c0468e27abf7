"""The drop-in claim against the reference's own types.

oracle/_ref/ref_dropin_check is compiled (oracle/Makefile) against the
unmodified reference headers and this repo's include/lance/b200.hpp.  It builds
reference lance::Tensor4 / FilterBank / ConvSpec / LanceConfig objects, runs
the reference's lance::lance_gemm (engines.hpp:492-536) and
lance::b200::lance_gemm_any on the SAME objects and compares the two
lance::Tensor4 results byte for byte; invalid specs / configs must raise
std::invalid_argument with the same message on both sides.

The binary is built here (where /root/reference exists) and travels to the GPU
box prebuilt; the reference tree itself does not.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "ref_dropin_check")


def _exe():
    if not os.path.exists(EXE) and os.path.isdir("/root/reference/proj/include"):
        from paper_2003_08646_b200 import _lib
        _lib.lib()  # the B200 library the check links against
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    if not os.path.exists(EXE):
        pytest.skip("oracle/_ref/ref_dropin_check not built (needs the reference headers)")
    return EXE


def test_validation_messages_match_reference():
    r = subprocess.run([_exe(), "--errors"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("errors same") == 8 and "ALL MATCH" in r.stdout


def test_no_cpu_fallback_through_reference_types():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("device present")
    r = subprocess.run([_exe()], capture_output=True, text=True, timeout=300)
    assert r.returncode == 1 and "no CPU fallback" in r.stderr


@pytest.mark.gpu
def test_reference_lance_gemm_vs_b200_same_objects():
    r = subprocess.run([_exe()], capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("-> bit-exact") == 10 and "ALL MATCH" in r.stdout
