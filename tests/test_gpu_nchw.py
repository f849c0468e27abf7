"""NCHW input option (north star: "coalesced 128-bit NCHW/NHWC loads"; the
reference is NHWC-only, tensor.hpp:24-55).  An NCHW plan reads x as
[N][C][H][W] through a device staging transpose; its codes, row sums,
parameters and NHWC output must be bit-identical to the NHWC path on the
transposed input and to the oracle (lance_gemm, engines.hpp:492-536) --
parity through a host transpose, SURVEY Appendix D.  Shapes cover ragged W / C
(the scalar transpose path), several 64-channel chunks and 32-pixel runs.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2003_08646_b200 as lance  # noqa: E402
from oracle import Oracle, Spec  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lo():
    return Oracle()


def cfg(bits_w=8, bits_i=8, gran=lance.Granularity.PerPosition):
    return lance.LanceConfig(bits_w, bits_i, gran, lance.LanceMode.Gemm)


def run(spec: Spec, x_nhwc, w, c, layout, params=None, stages=False):
    conv = lance.LanceConv(lance.ConvSpec(spec.n, spec.c, spec.h, spec.w, spec.k, spec.pad), c,
                           layout=layout)
    xin = x_nhwc if layout == "nhwc" else np.ascontiguousarray(x_nhwc.transpose(0, 3, 1, 2))
    xd = torch.from_numpy(np.ascontiguousarray(xin)).cuda()
    conv.set_filters(torch.from_numpy(w).cuda())
    y = conv.forward(xd, params=params)
    conv.sync()
    out = {"y": y.cpu().numpy()}
    if stages:
        for k in ("codes_a", "rowsum"):
            out[k] = conv.debug_read(k)
        out["params_a"] = lance.params_array(conv.params()[0])
    conv.close()
    return out


SHAPES = [
    Spec(2, 64, 16, 16, 32, 1),     # C = one chunk, W % 4 == 0 (128-bit loads)
    Spec(2, 40, 13, 11, 24, 1),     # ragged, W % 4 != 0 (scalar staging), C < 64
    Spec(1, 3, 32, 32, 16, 1),      # RGB
    Spec(2, 130, 10, 12, 48, 0),    # 3 channel chunks, pad 0
    Spec(1, 64, 100, 100, 16, 1),   # TW = 50: two 32/18-tile segments per tile row
    Spec(3, 128, 28, 28, 64, 1),    # ResNet R128 geometry (BK = 128, K1 row sums)
    Spec(2, 256, 14, 14, 64, 1),    # R256 geometry
]


@pytest.mark.parametrize("spec", SHAPES, ids=lambda s: f"n{s.n}c{s.c}h{s.h}w{s.w}k{s.k}p{s.pad}")
def test_nchw_matches_nhwc_and_oracle(lo, spec):
    x, w = lo.layer(spec, 17 + spec.c)
    c = cfg()
    a = run(spec, x, w, c, "nhwc", stages=True)
    b = run(spec, x, w, c, "nchw", stages=True)
    for k in ("codes_a", "rowsum", "params_a"):
        assert np.array_equal(a[k], b[k]), k
    assert np.array_equal(a["y"].view(np.uint32), b["y"].view(np.uint32))
    ref = lo.lance_gemm(spec, x, w)
    assert np.array_equal(b["y"].view(np.uint32), ref.view(np.uint32))


def test_nchw_pertensor_and_bits(lo):
    spec = Spec(2, 64, 18, 18, 32, 1)
    x, w = lo.layer(spec, 5)
    for c in (cfg(gran=lance.Granularity.PerTensor), cfg(4, 6)):
        b = run(spec, x, w, c, "nchw")
        ref = lo.lance_gemm(spec, x, w, bits_w=c.bits_w, bits_i=c.bits_i, gran=int(c.granularity))
        assert np.array_equal(b["y"].view(np.uint32), ref.view(np.uint32))


def test_nchw_static_params(lo):
    spec = Spec(2, 64, 16, 16, 32, 1)
    x, w = lo.layer(spec, 9)
    c = cfg()
    a = run(spec, x, w, c, "nhwc", stages=True)
    qp = [lance.QuantParams(8, float(t[1]), float(t[2]), float(t[3])) for t in a["params_a"]]
    # widen the ranges so some values clamp: static K1 path through NCHW staging
    qp = [lance.QuantParams(8, q.t_min * 0.5, q.t_max * 0.5, q.scale * 0.5) for q in qp]
    s1 = run(spec, x, w, c, "nhwc", params=qp)
    s2 = run(spec, x, w, c, "nchw", params=qp)
    assert np.array_equal(s1["y"].view(np.uint32), s2["y"].view(np.uint32))


@pytest.mark.slow
def test_nchw_resnet_r64_batch64(lo):
    """The R64 bench geometry (56x56, C = K = 64) at batch 64: 2-pass K0 over
    many CTA items, full-row segments (28 tiles), BN = 64 GEMM."""
    spec = Spec(64, 64, 56, 56, 64, 1)
    x, w = lo.layer(spec, 42)
    c = cfg()
    a = run(spec, x, w, c, "nhwc", stages=True)
    b = run(spec, x, w, c, "nchw", stages=True)
    for k in ("codes_a", "rowsum", "params_a"):
        assert np.array_equal(a[k], b[k]), k
    assert np.array_equal(a["y"].view(np.uint32), b["y"].view(np.uint32))


def test_nchw_f4(lo):
    """The staging transpose is layout-generic: NCHW also feeds F(4x4)."""
    spec = Spec(2, 64, 20, 20, 32, 1)
    x, w = lo.layer(spec, 3)
    c = cfg()
    conv = lance.LanceConv(lance.ConvSpec(2, 64, 20, 20, 32, 1), c, tile_m=4, layout="nchw")
    conv.set_filters(torch.from_numpy(w).cuda())
    y = conv.forward(torch.from_numpy(np.ascontiguousarray(x.transpose(0, 3, 1, 2))).cuda())
    conv.sync()
    ref = lo.lance_gemm(spec, x, w, tile_m=4)
    assert np.array_equal(y.cpu().numpy().view(np.uint32), ref.view(np.uint32))
    conv.close()


def test_nchw_rejects_bad_shapes(lo):
    spec = lance.ConvSpec(1, 8, 8, 8, 8, 1)
    conv = lance.LanceConv(spec, cfg(), layout="nchw")
    conv.set_filters(torch.zeros((8, 3, 3, 8), device="cuda"))
    with pytest.raises(lance.LanceError):
        conv.forward(torch.zeros((1, 8, 8, 8 + 1), device="cuda"))  # not [N, C, H, W]
    conv.close()
