"""CPU checks of the C-ABI boundary: the in-tree library loads and exports
every symbol include/lance_b200.h declares; validation mirrors the reference;
the UniformSource fixture matches the reference stream.  No compute calls."""
import ctypes as ct
import os
import re

import numpy as np
import pytest

import paper_2003_08646_b200 as lance
from paper_2003_08646_b200 import _lib
from oracle import Oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lance_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"LANCE_API\s+[\w\s\*]+?\b(lance_\w+)\s*\(", text)))


def test_header_declares_the_python_binding_set():
    assert declared_symbols() == sorted(_lib.EXPORTED)


def test_library_exports_every_declared_symbol():
    L = ct.CDLL(_lib.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(L, s)]
    assert not missing, missing
    assert _lib.lib().lance_abi_version() == 1


def test_cpp_header_declares_host_api():
    text = open(os.path.join(ROOT, "include", "lance", "b200.hpp")).read()
    for name in ("struct ConvSpec", "struct LanceConfig", "struct QuantParams", "struct Tensor4",
                 "struct FilterBank", "lance_gemm(", "class LanceConv"):
        assert name in text


@pytest.mark.parametrize("spec,cfg,msg", [
    (lance.ConvSpec(0, 1, 4, 4, 1), None, "all dims must be >= 1"),
    (lance.ConvSpec(1, 1, 4, 4, 1, pad=2), None, "pad must be 0 or 1"),
    (lance.ConvSpec(1, 1, 2, 2, 1, pad=0), None, "collapse to zero"),
    (lance.ConvSpec(1, 1, 4, 4, 1), lance.LanceConfig(9, 8, lance.Granularity.PerPosition,
                                                      lance.LanceMode.Gemm), "bits must be in"),
    (lance.ConvSpec(1, 1, 4, 4, 1), lance.LanceConfig(8, 8, lance.Granularity.PerTile,
                                                      lance.LanceMode.Gemm), "PerTile"),
    (lance.ConvSpec(1, 1, 4, 4, 1), lance.LanceConfig(8, 32, lance.Granularity.PerPosition,
                                                      lance.LanceMode.Gemm), "quantized operands"),
    (lance.ConvSpec(1, 1, 4, 4, 1), lance.LanceConfig(8, 8, lance.Granularity.PerPosition,
                                                      lance.LanceMode.Faithful), "mode must be Gemm"),
    (lance.ConvSpec(1, 32769, 4, 4, 1), None, "depth bound"),
])
def test_validation_mirrors_reference(spec, cfg, msg):
    cfg = cfg or lance.LanceConfig(8, 8, lance.Granularity.PerPosition, lance.LanceMode.Gemm)
    with pytest.raises(lance.LanceError, match=msg):
        lance.validate(spec, cfg)


def test_multiply_counts():
    s = lance.ConvSpec(1, 64, 32, 32, 64, 1)
    assert lance.winograd_multiply_count(s) == 16 * 256 * 64 * 64
    assert lance.direct_multiply_count(s) == 64 * 64 * 32 * 32 * 9
    s = lance.ConvSpec(256, 512, 7, 7, 512, 1)  # ragged: 4x4 tiles per 7x7 image
    assert lance.winograd_multiply_count(s) == 16 * 16 * 256 * 512 * 512


def test_multiply_counts_tiled():
    s = lance.ConvSpec(256, 64, 56, 56, 64, 1)
    assert lance.winograd_multiply_count_tiled(s, 2) == lance.winograd_multiply_count(s)
    assert lance.winograd_multiply_count_tiled(s, 4) == 36 * 14 * 14 * 256 * 64 * 64
    s = lance.ConvSpec(1, 8, 7, 7, 8, 1)  # 7x7 -> 2x2 tiles of 4
    assert lance.winograd_multiply_count_tiled(s, 4) == 36 * 4 * 8 * 8
    assert lance.winograd_multiply_count_tiled(s, 3) == 0


def test_uniform_fixture_matches_reference_stream():
    assert np.array_equal(lance.uniform_floats(4096, 42), Oracle().uniform(42, 4096))


def test_no_cpu_fallback_without_device():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("device present")
    s = lance.ConvSpec(1, 4, 8, 8, 4, 1)
    cfg = lance.LanceConfig(8, 8, lance.Granularity.PerPosition, lance.LanceMode.Gemm)
    with pytest.raises(lance.LanceDeviceError):
        lance.lance_gemm(np.zeros((1, 8, 8, 4), np.float32), np.zeros((4, 3, 3, 4), np.float32),
                         s, cfg)
    with pytest.raises(lance.LanceDeviceError):
        lance.lance_gemm(np.zeros((1, 8, 8, 4), np.float32), np.zeros((4, 3, 3, 4), np.float32),
                         s, cfg, tile_m=4)
