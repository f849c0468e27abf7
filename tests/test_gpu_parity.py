"""GPU parity of the B200 lance_gemm path against the reference (via the
golden digests and the pinned C oracle).  Integer stages (u8 codes, int32 row /
column sums, int32 accumulators) must be bit-exact; the fp32 output is checked
bitwise as well (tolerance 0 ULP; the north-star tolerance of rel-Frobenius
1e-6 is reported on failure).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2003_08646_b200 as lance  # noqa: E402
from oracle import Oracle, Spec  # noqa: E402
from tests.golden_cases import CASES, CASE_IDS, case_spec, digest, make_inputs  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lo():
    return Oracle()


def gemm_cfg(bits_w=8, bits_i=8, gran=1):
    return lance.LanceConfig(bits_w, bits_i, lance.Granularity(gran), lance.LanceMode.Gemm)


def to_spec(s: Spec) -> lance.ConvSpec:
    return lance.ConvSpec(s.n, s.c, s.h, s.w, s.k, s.pad)


def run_gpu(spec: Spec, x, w, cfg, acc=True, params=None):
    conv = lance.LanceConv(to_spec(spec), cfg)
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    wd = torch.from_numpy(np.ascontiguousarray(w)).cuda()
    accd = None
    if acc:
        accd = torch.empty((16, spec.rows, spec.k), dtype=torch.int32, device="cuda")
        conv.set_acc_dump(accd)
    conv.set_filters(wd)
    y = conv.forward(xd, params=params)
    conv.sync()
    out = {"y": y.cpu().numpy()}
    pa, pw = conv.params()
    out["params_a"] = lance.params_array(pa)
    out["params_w"] = lance.params_array(pw)
    for k in ("codes_a", "codes_w", "rowsum", "colsum"):
        out[k] = conv.debug_read(k)
    if acc:
        out["acc"] = accd.cpu().numpy()
    conv.close()
    return out


def mismatch_report(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    if a.dtype == np.float32:
        ai, bi = a.view(np.int32).astype(np.int64), b.view(np.int32).astype(np.int64)
        d = np.abs(ai - bi)
        rel = np.linalg.norm((a - b).astype(np.float64)) / max(np.linalg.norm(b.astype(np.float64)), 1e-30)
        return f"0-ULP {np.sum(d == 0)}, 1-ULP {np.sum(d == 1)}, >1-ULP {np.sum(d > 1)}, relF {rel:.3e}"
    d = np.abs(a.astype(np.int64) - b.astype(np.int64))
    return f"equal {np.sum(d == 0)}, 1-LSB {np.sum(d == 1)}, >1-LSB {np.sum(d > 1)}"


@pytest.mark.parametrize("case", CASES, ids=CASE_IDS)
def test_golden_stages_bitexact(lo, case):
    spec = case_spec(case)
    x, w = make_inputs(lo.uniform, spec, case["dist"], case["seed"])
    got = run_gpu(spec, x, w, gemm_cfg(case["bits_w"], case["bits_i"], case["gran"]))
    bad = [k for k, h in case["sha256"].items() if digest(got[k]) != h]
    if bad:
        _, ref = lo.lance_gemm(spec, x, w, bits_w=case["bits_w"], bits_i=case["bits_i"],
                               gran=case["gran"], dump=True)
        ref["y"] = lo.lance_gemm(spec, x, w, bits_w=case["bits_w"], bits_i=case["bits_i"],
                                 gran=case["gran"])
        msg = "; ".join(f"{k}: {mismatch_report(got[k], ref[k])}" for k in bad)
        pytest.fail(f"{case['name']} stages differ from the reference: {msg}")


def test_host_api_drop_in(lo):
    # lance_gemm(x, w, spec, cfg) on host arrays == reference, bitwise.
    spec = Spec(2, 64, 20, 20, 48, 1)
    x, w = make_inputs(lo.uniform, spec, "relu", 77)
    y = lance.lance_gemm(x, w, to_spec(spec), gemm_cfg())
    ref = lo.lance_gemm(spec, x, w)
    assert np.array_equal(y.view(np.uint32), ref.view(np.uint32)), mismatch_report(y, ref)
    # a second call reuses the cached plan and must give the same bits
    y2 = lance.lance_gemm(x, w, to_spec(spec), gemm_cfg())
    assert np.array_equal(y2.view(np.uint32), y.view(np.uint32))


@pytest.mark.parametrize("seed", range(6))
def test_random_shapes_vs_oracle(lo, seed):
    rng = np.random.default_rng(1000 + seed)
    spec = Spec(int(rng.integers(1, 4)), int(rng.integers(1, 80)), int(rng.integers(3, 24)),
                int(rng.integers(3, 24)), int(rng.integers(1, 80)), int(rng.integers(0, 2)))
    bw, bi, gran = int(rng.integers(2, 9)), int(rng.integers(2, 9)), int(rng.integers(1, 3))
    x, w = make_inputs(lo.uniform, spec, "relu" if seed % 2 else "uniform", seed)
    got = run_gpu(spec, x, w, gemm_cfg(bw, bi, gran))
    y, ref = lo.lance_gemm(spec, x, w, bits_w=bw, bits_i=bi, gran=gran, dump=True)
    ref["y"] = y
    for k in ("codes_a", "codes_w", "rowsum", "colsum", "acc", "params_a", "params_w", "y"):
        assert np.array_equal(np.asarray(got[k]).view(np.uint8), np.asarray(ref[k]).view(np.uint8)), \
            f"{spec} bits {bw}/{bi} gran {gran}: {k}: {mismatch_report(got[k], ref[k])}"


def test_nan_input_raises(lo):
    spec = Spec(1, 8, 10, 10, 8)
    x, w = make_inputs(lo.uniform, spec, "uniform", 3)
    x = x.copy()
    x[0, 4, 5, 2] = np.nan
    with pytest.raises(lance.LanceNaNError, match="NaN"):
        lance.lance_gemm(x, w, to_spec(spec), gemm_cfg())
    x[0, 4, 5, 2] = np.inf
    with pytest.raises(lance.LanceError):
        lance.lance_gemm(x, w, to_spec(spec), gemm_cfg())


def test_validation_matches_reference_messages():
    with pytest.raises(lance.LanceError, match="PerTile"):
        lance.LanceConv(lance.ConvSpec(1, 4, 8, 8, 4, 1),
                        lance.LanceConfig(mode=lance.LanceMode.Gemm))
    with pytest.raises(lance.LanceError, match="pad must be 0 or 1"):
        lance.LanceConv(lance.ConvSpec(1, 4, 8, 8, 4, 2), gemm_cfg())


def test_static_params_mode(lo):
    # Static params (no range pass): caller-provided QuantParams[16].
    spec = Spec(2, 32, 14, 14, 32, 1)
    x, w = make_inputs(lo.uniform, spec, "relu", 5)
    params = [lance.QuantParams(8, -1.5 - 0.1 * p, 2.0 + 0.05 * p,
                                np.float32((2.0 + 0.05 * p + 1.5 + 0.1 * p) / 255.0))
              for p in range(16)]
    arr = lance.params_array(params)
    got = run_gpu(spec, x, w, gemm_cfg(), params=params)
    y, ref = lo.lance_gemm(spec, x, w, in_params=arr, dump=True)
    assert np.array_equal(got["codes_a"], ref["codes_a"])
    assert np.array_equal(got["acc"], ref["acc"])
    assert np.array_equal(got["y"].view(np.uint32), y.view(np.uint32)), mismatch_report(got["y"], y)


def test_bias_relu_epilogue(lo):
    spec = Spec(1, 16, 12, 12, 24, 1)
    x, w = make_inputs(lo.uniform, spec, "uniform", 8)
    bias = lo.uniform(99, spec.k)
    conv = lance.LanceConv(to_spec(spec), gemm_cfg())
    conv.set_filters(torch.from_numpy(w).cuda())
    conv.set_epilogue(torch.from_numpy(bias).cuda(), relu=True)
    y = conv.forward(torch.from_numpy(x).cuda())
    conv.sync()
    ref = lo.lance_gemm(spec, x, w)
    exp = np.maximum(ref + bias.reshape(1, 1, 1, -1), np.float32(0)) + np.float32(0)
    assert np.array_equal(y.cpu().numpy().view(np.uint32), exp.view(np.uint32))


def test_launch_count_and_native_library():
    import os
    spec = lance.ConvSpec(1, 64, 32, 32, 64, 1)
    conv = lance.LanceConv(spec, gemm_cfg())
    conv.set_filters(torch.randn(64, 3, 3, 64, device="cuda"))
    conv.forward(torch.randn(1, 32, 32, 64, device="cuda"))
    conv.sync()
    assert conv.last_launch_count == 3
    maps = open("/proc/self/maps").read()
    assert "liblance_b200.so" in maps


def test_global_params_across_shards(lo):
    # SURVEY 8(e) mode 2 on one device: two batch shards each run the range
    # pass, their (min, max) are combined (what the 128-byte all-reduce does
    # across GPUs), and both shards quantise with the full-batch params: the
    # concatenated output equals one full-batch reference call bitwise.
    from paper_2003_08646_b200 import shard
    spec = Spec(4, 64, 14, 14, 32, 1)
    x, w = make_inputs(lo.uniform, spec, "relu", 41)
    wd = torch.from_numpy(w).cuda()
    convs, los, his = [], [], []
    for r in range(2):
        a, b = shard.shard_range(spec.n, 2, r)
        c = lance.LanceConv(lance.ConvSpec(b - a, spec.c, spec.h, spec.w, spec.k, 1), gemm_cfg())
        c.set_filters(wd)
        c.forward(torch.from_numpy(np.ascontiguousarray(x[a:b])).cuda())
        c.sync()
        pa, _ = c.params()
        los.append([q.t_min for q in pa])
        his.append([q.t_max for q in pa])
        convs.append((c, a, b))
    params = shard.params_from_minmax(np.min(los, axis=0), np.max(his, axis=0), 8)
    ys = []
    for c, a, b in convs:
        y = c.forward(torch.from_numpy(np.ascontiguousarray(x[a:b])).cuda(), params=params)
        c.sync()
        ys.append(y.cpu().numpy())
    got = np.concatenate(ys)
    ref = lo.lance_gemm(spec, x, w)
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32)), mismatch_report(got, ref)


@pytest.mark.parametrize("spec,dist,seed", [(Spec(2, 64, 17, 17, 64, 1), "relu", 3),   # row sums in the GEMM
                                            (Spec(1, 128, 14, 14, 64, 1), "uniform", 4),  # row sums in K1
                                            (Spec(1, 256, 9, 9, 128, 0), "relu", 5),
                                            (Spec(3, 3, 15, 13, 20, 1), "relu", 6)],      # small-C kernels
                         ids=lambda v: str(v))
def test_kernel_family_shapes_bitexact(lo, spec, dist, seed):
    # One shape per input-kernel family / row-sum placement, every stage bitwise.
    x, w = make_inputs(lo.uniform, spec, dist, seed)
    got = run_gpu(spec, x, w, gemm_cfg())
    y, ref = lo.lance_gemm(spec, x, w, dump=True)
    ref["y"] = y
    for k in ("codes_a", "rowsum", "acc", "params_a", "y"):
        assert np.array_equal(np.asarray(got[k]).view(np.uint8), np.asarray(ref[k]).view(np.uint8)), \
            f"{spec}: {k}: {mismatch_report(got[k], ref[k])}"


def test_tensor_shape_checked():
    # check_layer (engines.hpp:84-91): an NCHW input or a [K,C,3,3] filter bank
    # with the right element count is rejected, like the reference.
    spec = lance.ConvSpec(1, 4, 6, 6, 8, 1)
    conv = lance.LanceConv(spec, gemm_cfg())
    with pytest.raises(lance.LanceError, match="filter dims do not match spec"):
        conv.set_filters(torch.zeros(8, 4, 3, 3, device="cuda"))
    conv.set_filters(torch.zeros(8, 3, 3, 4, device="cuda"))
    with pytest.raises(lance.LanceError, match="input tensor dims do not match spec"):
        conv.forward(torch.zeros(1, 4, 6, 6, device="cuda"))
    conv.close()


def test_large_k_layer(lo):
    # K = 2048 filters (32 n-tiles): the epilogue's third-term table is per
    # tile, so shared memory no longer grows with K.
    spec = Spec(1, 64, 6, 6, 2048, 1)
    x, w = make_inputs(lo.uniform, spec, "relu", 12)
    got = run_gpu(spec, x, w, gemm_cfg(), acc=False)
    ref = lo.lance_gemm(spec, x, w)
    assert np.array_equal(got["y"].view(np.uint32), ref.view(np.uint32)), mismatch_report(got["y"], ref)


@pytest.mark.parametrize("spec", [Spec(2, 64, 17, 17, 64, 1),    # fast K1, row sums in the GEMM
                                  Spec(1, 128, 14, 14, 64, 1),   # fast K1, row sums in K1
                                  Spec(1, 96, 9, 11, 24, 0)])    # generic K1
def test_static_params_out_of_range_bitexact(lo, spec):
    """Static (caller) params narrower than / shifted from the data: codes
    saturate at 0 and top, one position has scale 0 -- the fast static
    quantiser's clamps and tie fallback must reproduce quantize() exactly."""
    x, w = make_inputs(lo.uniform, spec, "relu", 41)
    _, d = lo.lance_gemm(spec, x, w, dump=True)
    pa = d["params_a"].copy()
    rng = np.random.default_rng(0)
    for p in range(16):
        lo_, hi_ = float(pa[p, 1]), float(pa[p, 2])
        span = hi_ - lo_
        a = np.float32(lo_ + span * rng.uniform(0.1, 0.4))
        b = np.float32(hi_ - span * rng.uniform(0.1, 0.4))
        pa[p, 1], pa[p, 2] = a, b
        pa[p, 3] = np.float32(np.float32(b - a) / np.float32(255.0))
    pa[5, 2] = pa[5, 1]
    pa[5, 3] = np.float32(0.0)  # scale 0 -> every code 0
    qps = [lance.QuantParams(8, float(r[1]), float(r[2]), float(r[3])) for r in pa]
    got = run_gpu(spec, x, w, gemm_cfg(), params=qps)
    y, ref = lo.lance_gemm(spec, x, w, in_params=pa, dump=True)
    ref["y"] = y
    for k in ("codes_a", "rowsum", "acc", "y"):
        assert np.array_equal(np.asarray(got[k]).view(np.uint8), np.asarray(ref[k]).view(np.uint8)), \
            f"{k}: {mismatch_report(got[k], ref[k])}"


@pytest.mark.parametrize("tile_m", [2, 4])
def test_device_ranges_across_shards(lo, tile_m):
    # Global-fit mode through the device API (lance_plan_ranges ->
    # element-wise MAX of the [-t_min, t_max, nan] buffers, what the NCCL
    # all-reduce does across GPUs -> lance_plan_forward_ranges): the shards'
    # outputs concatenate to one full-batch reference call bitwise.
    spec = Spec(5, 64, 14, 14, 48, 1)
    x, w = make_inputs(lo.uniform, spec, "relu", 43)
    wd = torch.from_numpy(w).cuda()
    from paper_2003_08646_b200 import shard
    convs, bufs = [], []
    for r in range(2):
        a, b = shard.shard_range(spec.n, 2, r)
        c = lance.LanceConv(lance.ConvSpec(b - a, spec.c, spec.h, spec.w, spec.k, 1), gemm_cfg(),
                            tile_m=tile_m)
        c.set_filters(wd)
        xs = torch.from_numpy(np.ascontiguousarray(x[a:b])).cuda()
        bufs.append(c.ranges(xs))
        convs.append((c, xs))
    g = torch.maximum(bufs[0], bufs[1])
    ys = []
    for c, xs in convs:
        ys.append(c.forward(xs, ranges=g))
        c.sync()
    got = torch.cat(ys).cpu().numpy()
    ref = lo.lance_gemm(spec, x, w, tile_m=tile_m)
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32)), mismatch_report(got, ref)
    # a NaN on one shard is reported by every shard's forward (the reference
    # throws from fit_params over the whole batch, quant.hpp:62)
    xb = x[:3].copy()  # shard 0 holds images 0..2
    xb[1, 3, 3, 5] = np.nan
    c0, xs0 = convs[0]
    bad = c0.ranges(torch.from_numpy(xb).cuda())
    g2 = torch.maximum(bad, bufs[1])
    c1, xs1 = convs[1]
    c1.forward(xs1, ranges=g2)
    with pytest.raises(lance.LanceNaNError):
        c1.sync()
    for c, _ in convs:
        c.close()
