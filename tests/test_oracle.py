"""CPU tests pinning the oracle (the parity checker of the B200 path).

The C restatement (oracle/lance_oracle.c) is checked against
  * the reference's own known-answer tests (test_quant.cpp, test_winograd.cpp),
  * the golden digests generated from the reference (tests/golden/golden.json),
  * the reference compiled in place (oracle/_ref), when it is present.
"""
import math

import numpy as np
import pytest

import oracle
from oracle import Oracle, Spec, OracleError
from tests.golden_cases import CASES, CASE_IDS, case_spec, digest, make_inputs


@pytest.fixture(scope="module")
def lo():
    return Oracle()


@pytest.fixture(scope="module")
def ref():
    if not oracle.reference_available():
        pytest.skip("reference shim not built (reference tree absent)")
    return oracle.Reference()


# --- reference known-answer tests (test_quant.cpp:36-94) ------------------

def test_fit_params_ramp_2bit(lo):
    p = lo.fit_params(np.arange(16, dtype=np.float32), 2)
    assert (p.t_min, p.t_max, p.scale) == (0.0, 15.0, 5.0)


def test_fit_params_degenerate_and_two_point(lo):
    p = lo.fit_params([7.5], 8)
    assert (p.t_min, p.t_max, p.scale) == (7.5, 7.5, 0.0)
    q = lo.fit_params([-1.0, 1.0], 8)
    assert math.isclose(q.scale, 2.0 / 255.0, rel_tol=1e-7)


def test_fit_params_rejects(lo):
    with pytest.raises(OracleError):
        lo.fit_params(np.zeros(0, np.float32), 8)
    with pytest.raises(OracleError):
        lo.fit_params(np.arange(16), 1)
    with pytest.raises(OracleError):
        lo.fit_params(np.arange(16), 9)
    with pytest.raises(OracleError, match="NaN"):
        lo.fit_params([1.0, float("nan")], 8)


def test_quantize_ramp_table(lo):
    p = lo.fit_params(np.arange(16, dtype=np.float32), 2)
    expected = [0, 0, 0, 1, 1, 1, 1, 1, 2, 2, 2, 2, 2, 3, 3, 3]
    assert [lo.quantize(float(i), p) for i in range(16)] == expected
    assert lo.quantize(7.0, p) == 1
    assert lo.quantize(-100.0, p) == 0 and lo.quantize(1000.0, p) == 3
    d = lo.fit_params([4.0], 4)
    assert lo.quantize(4.0, d) == 0 and lo.quantize(123.0, d) == 0


def test_dequantize_grid(lo):
    p = lo.fit_params(np.arange(16, dtype=np.float32), 2)
    assert [lo.dequantize(c, p) for c in (0, 1, 3)] == [0.0, 5.0, 15.0]


# --- transforms (test_winograd.cpp:68-146) --------------------------------

def test_input_transform_golden_eq6(lo):
    d = np.array([[0, 1, 1, 1], [1, 1, 2, 2], [2, 2, 2, 3], [3, 3, 3, 3]], np.float32)
    exp = np.array([[-1, -2, 0, 1], [-1, 7, 1, -2], [1, 1, -1, 0], [-1, -3, 1, -1]], np.float32)
    assert np.array_equal(lo.transform_input(d), exp)


def test_filter_transform_kats(lo):
    exp = np.array([[1, 1.5, .5, 1], [1.5, 2.25, .75, 1.5], [.5, .75, .25, .5],
                    [1, 1.5, .5, 1]], np.float32)
    assert np.array_equal(lo.transform_filter(np.ones((3, 3))), exp)
    c = np.zeros((3, 3)); c[1, 1] = 1
    col = np.array([0, .5, -.5, 0], np.float32)
    assert np.array_equal(lo.transform_filter(c), np.outer(col, col))
    k = np.zeros((3, 3)); k[0, 0] = 1
    col0 = np.array([1, .5, .5, 0], np.float32)
    assert np.array_equal(lo.transform_filter(k), np.outer(col0, col0))


def test_output_transform_ones(lo):
    assert np.array_equal(lo.transform_output(np.ones((4, 4))), [[9, -3], [-3, 1]])


def test_never_negative_zero(lo):
    # matrix.hpp:75-84 accumulates from +0.0f, so -0.0 inputs give +0.0.
    v = lo.transform_input(np.full((4, 4), -0.0, np.float32))
    assert not np.any(np.signbit(v))


# --- validation (engines.hpp:46-91, 496-499) ------------------------------

@pytest.mark.parametrize("spec,kw,msg", [
    (Spec(0, 1, 4, 4, 1), {}, "all dims must be >= 1"),
    (Spec(1, 1, 4, 4, 1, pad=2), {}, "pad must be 0 or 1"),
    (Spec(1, 1, 2, 2, 1, pad=0), {}, "collapse to zero"),
    (Spec(1, 1, 4, 4, 1), {"bits_w": 9}, "bits must be in"),
    (Spec(1, 1, 4, 4, 1), {"gran": 0}, "PerTile"),
    (Spec(1, 1, 4, 4, 1), {"bits_i": 32}, "quantized operands"),
    (Spec(1, 1, 4, 4, 1), {"mode_gemm": False}, "mode must be Gemm"),
    (Spec(1, 32769, 4, 4, 1), {}, "depth bound"),
])
def test_validation_messages(lo, spec, kw, msg):
    with pytest.raises(OracleError, match=msg):
        lo.validate(spec, **kw)


# --- golden digests (generated from the reference) ------------------------

@pytest.mark.parametrize("case", CASES, ids=CASE_IDS)
def test_oracle_matches_golden(lo, case):
    spec = case_spec(case)
    x, w = make_inputs(lo.uniform, spec, case["dist"], case["seed"])
    y, st = lo.lance_gemm(spec, x, w, bits_w=case["bits_w"], bits_i=case["bits_i"],
                          gran=case["gran"], dump=True)
    st["y"] = y
    for k, h in case["sha256"].items():
        assert digest(st[k]) == h, f"{case['name']}: stage {k} differs from the reference"


# --- live reference ---------------------------------------------------------

def test_reference_property_suite(ref):
    ok, report = ref.run_verify()
    assert ok, report


def test_uniform_stream_matches_reference(lo, ref):
    assert np.array_equal(lo.uniform(12345, 5000), ref.uniform(12345, 5000))


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_oracle_matches_reference_random_shapes(lo, ref, seed):
    rng = np.random.default_rng(seed)
    for _ in range(4):
        spec = Spec(int(rng.integers(1, 3)), int(rng.integers(1, 20)), int(rng.integers(3, 13)),
                    int(rng.integers(3, 13)), int(rng.integers(1, 20)), int(rng.integers(0, 2)))
        bw, bi = int(rng.integers(2, 9)), int(rng.integers(2, 9))
        gran = int(rng.integers(1, 3))
        x, w = make_inputs(lo.uniform, spec, "relu" if seed % 2 else "uniform", seed + 100)
        y0 = ref.lance_gemm(spec, x, w, bits_w=bw, bits_i=bi, gran=gran)
        y1 = lo.lance_gemm(spec, x, w, bits_w=bw, bits_i=bi, gran=gran)
        assert np.array_equal(y0.view(np.uint32), y1.view(np.uint32))


def test_nan_input_rejected_like_reference(lo, ref):
    spec = Spec(1, 4, 6, 6, 2)
    x, w = make_inputs(lo.uniform, spec, "uniform", 3)
    x = x.copy(); x[0, 2, 3, 1] = np.nan
    with pytest.raises(OracleError, match="NaN"):
        ref.lance_gemm(spec, x, w)
    with pytest.raises(OracleError, match="NaN"):
        lo.lance_gemm(spec, x, w)


def test_gemm_mode_equivalence_c1_bitwise(ref):
    # engines.hpp:488-491: lance_gemm == lance_faithful exactly at C = 1.
    spec = Spec(2, 1, 8, 8, 3)
    o = Oracle()
    x, w = make_inputs(o.uniform, spec, "uniform", 17)
    a = ref.lance_gemm(spec, x, w)
    b = ref.lance_faithful(spec, x, w)
    assert np.array_equal(a, b)
