"""F(4x4,3x3) extension (BASELINE config 4).

The reference ships F(2x2,3x3) only (winograd.hpp:27; extract_tiles
tensor.hpp:117-118 rejects m != 2), so this path's oracle is the reference
algorithm re-run with the Appendix D basis (oracle lo_lance_gemm_tiled,
tile_m = 4), evaluated in the reference's matmul order (matrix.hpp:75-84).
Parity here is SELF-PINNED, in three independent ways:
  * the basis: the correlation identity of verify.hpp:147-166, for 6x6 tiles;
  * the glue: every stage of the oracle's F(4x4) run is recomposed from the
    primitive transforms, fit_params / quantize and integer GEMMs, bitwise;
  * drift: digests in tests/golden/golden_f4.json (make_golden_f4.py).
The GPU F(4x4) kernels are checked against this oracle bitwise
(tests/test_gpu_f4.py).
"""
import json
import os

import numpy as np
import pytest

from oracle import Oracle, Spec
from tests.golden.make_golden import digest, make_inputs

HERE = os.path.dirname(os.path.abspath(__file__))
with open(os.path.join(HERE, "golden", "golden_f4.json")) as f:
    GOLDEN_F4 = json.load(f)["cases"]


@pytest.fixture(scope="module")
def lo():
    return Oracle()


def test_f4_correlation_identity(lo):
    """verify.hpp:147-166 pattern for F(4x4): A^T[(G g G^T) .* (B^T d B)]A equals
    the 3x3 correlation of a 6x6 tile (fp32; measured worst 1.1e-5)."""
    rng = np.random.default_rng(101)
    worst = 0.0
    for _ in range(1000):
        d = rng.uniform(-1, 1, (6, 6)).astype(np.float32)
        g = rng.uniform(-1, 1, (3, 3)).astype(np.float32)
        via = lo.transform_output4(lo.transform_filter4(g) * lo.transform_input4(d))
        ref = np.zeros((4, 4))
        for r in range(3):
            for s in range(3):
                ref += d[r:r + 4, s:s + 4].astype(np.float64) * float(g[r, s])
        worst = max(worst, float(np.abs(via - ref).max()))
    assert worst < 5e-5, worst


def test_f4_transforms_match_matmul_order(lo):
    """The C transforms are (T x) T^T with the i-k-j fp32 accumulation from +0 of
    matrix.hpp:75-84, restated here in numpy float32 scalar steps."""
    def matmul(a, b):
        out = np.zeros((a.shape[0], b.shape[1]), np.float32)
        for i in range(a.shape[0]):
            for k in range(a.shape[1]):
                for j in range(b.shape[1]):
                    out[i, j] = np.float32(out[i, j] + np.float32(a[i, k] * b[k, j]))
        return out
    f = np.float32
    bt = np.array([[4, 0, -5, 0, 1, 0], [0, -4, -4, 1, 1, 0], [0, 4, -4, -1, 1, 0],
                   [0, -2, -1, 2, 1, 0], [0, 2, -1, -2, 1, 0], [0, 4, 0, -5, 0, 1]], np.float32)
    g6 = np.array([[0.25, 0, 0], [-f(1) / f(6)] * 3, [-f(1) / f(6), f(1) / f(6), -f(1) / f(6)],
                   [f(1) / f(24), f(1) / f(12), f(1) / f(6)], [f(1) / f(24), -f(1) / f(12), f(1) / f(6)],
                   [0, 0, 1]], np.float32)
    at = np.array([[1, 1, 1, 1, 1, 0], [0, 1, -1, 2, -2, 0], [0, 1, 1, 4, 4, 0],
                   [0, 1, -1, 8, -8, 1]], np.float32)
    rng = np.random.default_rng(5)
    for _ in range(20):
        d = rng.uniform(-1, 1, (6, 6)).astype(np.float32)
        g = rng.uniform(-1, 1, (3, 3)).astype(np.float32)
        m = rng.uniform(-3, 3, (6, 6)).astype(np.float32)
        assert np.array_equal(lo.transform_input4(d), matmul(matmul(bt, d), bt.T))
        assert np.array_equal(lo.transform_filter4(g), matmul(matmul(g6, g), g6.T))
        assert np.array_equal(lo.transform_output4(m), matmul(matmul(at, m), at.T))


@pytest.mark.parametrize("spec,dist", [(Spec(2, 5, 11, 9, 3, 1), "relu"),
                                       (Spec(1, 4, 8, 10, 2, 0), "uniform")])
def test_f4_pipeline_recomposes_bitwise(lo, spec, dist):
    """Every stage of lance_gemm(tile_m=4) rebuilt from the primitives: tiles of
    side 6 at stride 4 (zero padded), per-position fit_params + quantize, the
    36 integer GEMMs with row/col sums, affine_term, A^T m A and the merge."""
    x, w = make_inputs(lo.uniform, spec, dist, 17)
    y, st = lo.lance_gemm(spec, x, w, dump=True, tile_m=4)
    OH, OW = spec.out_h, spec.out_w
    TH, TW = (OH + 3) // 4, (OW + 3) // 4
    M, C, K = spec.rows_m(4), spec.c, spec.k
    assert st["v"].shape == (36, M, C)
    xp = np.zeros((spec.n, spec.h + 2 * spec.pad + 8, spec.w + 2 * spec.pad + 8, C), np.float32)
    xp[:, spec.pad:spec.pad + spec.h, spec.pad:spec.pad + spec.w] = x
    for img in range(spec.n):
        for ti in range(TH):
            for tj in range(TW):
                row = (img * TH + ti) * TW + tj
                for c in range(C):
                    d = xp[img, 4 * ti:4 * ti + 6, 4 * tj:4 * tj + 6, c]
                    assert np.array_equal(st["v"][:, row, c], lo.transform_input4(d).ravel())
    for k in range(K):
        for c in range(C):
            assert np.array_equal(st["u"][:, c, k], lo.transform_filter4(w[k, :, :, c]).ravel())
    pa, pw = [], []
    for p in range(36):
        qa = lo.fit_params(st["v"][p], 8)
        qw = lo.fit_params(st["u"][p], 8)
        assert (qa.t_min, qa.t_max, qa.scale) == tuple(st["params_a"][p][1:])
        pa.append(qa)
        pw.append(qw)
        for i, val in enumerate(st["v"][p].ravel()[:200]):
            assert st["codes_a"][p].ravel()[i] == lo.quantize(val, qa)
    A = st["codes_a"].astype(np.int64)
    B = st["codes_w"].astype(np.int64)
    assert np.array_equal(st["acc"], np.einsum("pmc,pck->pmk", A, B).astype(np.int32))
    assert np.array_equal(st["rowsum"], A.sum(axis=2).astype(np.int32))
    assert np.array_equal(st["colsum"], B.sum(axis=1).astype(np.int32))
    for row in range(M):
        img, t = divmod(row, TH * TW)
        ti, tj = divmod(t, TW)
        for k in range(K):
            mdom = np.array([lo.affine_term(int(st["acc"][p, row, k]), int(st["rowsum"][p, row]),
                                            int(st["colsum"][p, k]), C, pa[p], pw[p])
                             for p in range(36)], np.float32)
            s = lo.transform_output4(mdom)
            for a in range(4):
                for b in range(4):
                    oi, oj = 4 * ti + a, 4 * tj + b
                    if oi < OH and oj < OW:
                        assert y[img, oi, oj, k].view(np.uint32) == s[a, b].view(np.uint32)


@pytest.mark.parametrize("spec", [Spec(2, 16, 12, 12, 8, 1), Spec(2, 32, 13, 11, 16, 0)])
def test_f4_error_vs_direct(lo, spec):
    """8-bit LANCE F(4x4) vs the fp32 direct conv: relative Frobenius error
    below 0.15 (measured 0.07-0.09; F(2x2) measures 0.013 on the same layers --
    the wider F(4x4) transform range costs quantization resolution)."""
    x, w = make_inputs(lo.uniform, spec, "relu", 5)
    yd = lo.direct_conv(spec, x, w)
    y4 = lo.lance_gemm(spec, x, w, tile_m=4)
    y2 = lo.lance_gemm(spec, x, w, tile_m=2)
    e4 = np.linalg.norm(y4 - yd) / np.linalg.norm(yd)
    e2 = np.linalg.norm(y2 - yd) / np.linalg.norm(yd)
    assert e4 < 0.15 and e2 < e4


def test_tile_m_2_is_the_reference_path(lo):
    spec = Spec(2, 16, 9, 7, 8, 1)
    x, w = make_inputs(lo.uniform, spec, "relu", 3)
    assert np.array_equal(lo.lance_gemm(spec, x, w, tile_m=2), lo.lance_gemm(spec, x, w))


@pytest.mark.parametrize("case", GOLDEN_F4, ids=[c["name"] for c in GOLDEN_F4])
def test_f4_oracle_matches_golden(lo, case):
    spec = Spec(*case["spec"])
    x, w = make_inputs(lo.uniform, spec, case["dist"], case["seed"])
    y, st = lo.lance_gemm(spec, x, w, bits_w=case["bits_w"], bits_i=case["bits_i"],
                          gran=case["gran"], dump=True, tile_m=4)
    st["y"] = y
    for k, h in case["sha256"].items():
        assert digest(st[k]) == h, k
