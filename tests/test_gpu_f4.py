"""GPU parity of the F(4x4,3x3) extension (paper_2003_08646_b200/csrc/lance_f4.cu)
against the oracle's lo_lance_gemm_tiled(tile_m=4) (self-pinned; see
tests/test_f4.py) and the committed digests tests/golden/golden_f4.json.
Integer stages (u8 codes, int32 row / column sums, int32 accumulators) and the
fp32 output are compared bitwise (tolerance 0)."""
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2003_08646_b200 as lance  # noqa: E402
from oracle import Oracle, Spec  # noqa: E402
from tests.golden.make_golden import digest, make_inputs  # noqa: E402
from tests.test_gpu_parity import gemm_cfg, mismatch_report, to_spec  # noqa: E402

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
with open(os.path.join(HERE, "golden", "golden_f4.json")) as f:
    GOLDEN_F4 = json.load(f)["cases"]


@pytest.fixture(scope="module")
def lo():
    return Oracle()


def run_gpu_f4(spec: Spec, x, w, cfg, params=None, bias=None, relu=False):
    conv = lance.LanceConv(to_spec(spec), cfg, tile_m=4)
    assert conv.positions == 36
    M = spec.rows_m(4)
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    wd = torch.from_numpy(np.ascontiguousarray(w)).cuda()
    accd = torch.empty((36, M, spec.k), dtype=torch.int32, device="cuda")
    conv.set_acc_dump(accd)
    if bias is not None or relu:
        conv.set_epilogue(torch.from_numpy(bias).cuda() if bias is not None else None, relu)
    conv.set_filters(wd)
    y = conv.forward(xd, params=params)
    conv.sync()
    out = {"y": y.cpu().numpy(), "acc": accd.cpu().numpy()}
    pa, pw = conv.params()
    out["params_a"] = lance.params_array(pa)
    out["params_w"] = lance.params_array(pw)
    for k in ("codes_a", "codes_w", "rowsum", "colsum"):
        out[k] = conv.debug_read(k)
    conv.close()
    return out


def compare(got, ref, keys):
    bad = [k for k in keys if not np.array_equal(np.asarray(got[k]).view(np.uint8),
                                                 np.asarray(ref[k]).view(np.uint8))]
    return "; ".join(f"{k}: {mismatch_report(got[k], ref[k])}" for k in bad)


@pytest.mark.parametrize("case", GOLDEN_F4, ids=[c["name"] for c in GOLDEN_F4])
def test_f4_golden_stages_bitexact(lo, case):
    spec = Spec(*case["spec"])
    x, w = make_inputs(lo.uniform, spec, case["dist"], case["seed"])
    got = run_gpu_f4(spec, x, w, gemm_cfg(case["bits_w"], case["bits_i"], case["gran"]))
    bad = [k for k, h in case["sha256"].items() if digest(got[k]) != h]
    if bad:
        y, ref = lo.lance_gemm(spec, x, w, bits_w=case["bits_w"], bits_i=case["bits_i"],
                               gran=case["gran"], dump=True, tile_m=4)
        ref["y"] = y
        pytest.fail(f"{case['name']}: {compare(got, ref, bad)}")


@pytest.mark.parametrize("spec", [
    Spec(2, 64, 28, 28, 64, 1),     # BK 64, 4 n-tiles, several row blocks
    Spec(1, 128, 14, 14, 128, 1),   # BK 128
    Spec(3, 96, 13, 9, 24, 0),      # BK 32, ragged tiles, K not a multiple of 16
    Spec(1, 512, 7, 7, 512, 1),     # ResNet-18 R512 slice: 32 n-tiles, C*255^2 >= 2^24 (I2F epilogue)
])
def test_f4_shapes_bitexact(lo, spec):
    x, w = make_inputs(lo.uniform, spec, "relu", 23)
    got = run_gpu_f4(spec, x, w, gemm_cfg())
    y, ref = lo.lance_gemm(spec, x, w, dump=True, tile_m=4)
    ref["y"] = y
    msg = compare(got, ref, ("codes_a", "rowsum", "codes_w", "colsum", "acc", "params_a",
                             "params_w", "y"))
    assert not msg, msg


def test_f4_static_params_bitexact(lo):
    """Caller-supplied 36 input params (no range pass): quantiser with values
    outside [t_min, t_max], exact division path."""
    spec = Spec(2, 32, 12, 12, 16, 1)
    x, w = make_inputs(lo.uniform, spec, "uniform", 9)
    _, d = lo.lance_gemm(spec, x, w, dump=True, tile_m=4)
    pa = d["params_a"].copy()
    pa[:, 1] *= np.float32(0.5)   # narrower ranges: saturating codes
    pa[:, 2] *= np.float32(0.5)
    pa[:, 3] = ((pa[:, 2] - pa[:, 1]) / np.float32(255.0)).astype(np.float32)
    qps = [lance.QuantParams(8, float(r[1]), float(r[2]), float(r[3])) for r in pa]
    got = run_gpu_f4(spec, x, w, gemm_cfg(), params=qps)
    y, ref = lo.lance_gemm(spec, x, w, in_params=pa, dump=True, tile_m=4)
    ref["y"] = y
    msg = compare(got, ref, ("codes_a", "rowsum", "acc", "y"))
    assert not msg, msg


def test_f4_bias_relu_epilogue(lo):
    spec = Spec(2, 32, 10, 10, 20, 1)
    x, w = make_inputs(lo.uniform, spec, "relu", 4)
    bias = lo.uniform(77, spec.k).astype(np.float32)
    got = run_gpu_f4(spec, x, w, gemm_cfg(), bias=bias, relu=True)
    y = lo.lance_gemm(spec, x, w, tile_m=4)
    expect = np.maximum(y + bias, np.float32(0.0)) + np.float32(0.0)
    assert np.array_equal(got["y"].view(np.uint32), expect.view(np.uint32))


def test_f4_host_api(lo):
    spec = Spec(2, 16, 11, 11, 8, 1)
    x, w = make_inputs(lo.uniform, spec, "uniform", 12)
    cfg = gemm_cfg()
    y = lance.lance_gemm(x, w, to_spec(spec), cfg, tile_m=4)
    assert np.array_equal(y.view(np.uint32), lo.lance_gemm(spec, x, w, tile_m=4).view(np.uint32))
    # the tile_m = 2 host path is unchanged
    y2 = lance.lance_gemm(x, w, to_spec(spec), cfg)
    assert np.array_equal(y2.view(np.uint32), lo.lance_gemm(spec, x, w).view(np.uint32))


def test_f4_nan_reported(lo):
    spec = Spec(1, 8, 8, 8, 4, 1)
    x, w = make_inputs(lo.uniform, spec, "uniform", 3)
    x[0, 3, 3, 2] = np.nan
    with pytest.raises(lance.LanceNaNError):
        lance.lance_gemm(x, w, to_spec(spec), gemm_cfg(), tile_m=4)
