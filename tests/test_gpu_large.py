"""Config-5 extremes (BASELINE.json configs[4]: C, K in {64..512}, H = W in
{7..112}, batch 1..1024) at full size, checked the way SURVEY.md section 8(c)
"Large shapes" prescribes: the batch-coupled parameters are verified against an
exact host recomputation over the WHOLE batch, and the outputs on batch slices
through the pinned oracle with those parameters (images are independent given
the batch's QuantParams, engines.hpp:199-200; static-params oracle path).

* params: v = B^T d B for every tile and channel, evaluated in float32 numpy in
  the reference's column-first order (winograd.hpp:40-84, matrix.hpp:75-84),
  per-position min / max folded over the batch in image chunks, then the
  oracle's fit_params (quant.hpp:54-72) -- must equal the GPU's fitted input
  QuantParams bit for bit;
* y: first, middle and last images, oracle lance_gemm with the GPU's params
  (in_params) -- bitwise; every output of the batch finite.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2003_08646_b200 as lance  # noqa: E402
from oracle import Oracle, Spec  # noqa: E402

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

LARGE = [
    (1024, 64, 64, 56),    # batch 1024 (M = 802,816 rows, x = 822 MB)
    (64, 64, 64, 112),     # H = 112
    (1024, 512, 512, 7),   # batch 1024 at C = K = 512
    (4, 512, 512, 112),    # C = K = 512 at H = 112
    (64, 128, 512, 28),    # C != K
]


def v_ranges(x, pad, chunk=16):
    """Per-position (min, max) of v = B^T d B over all tiles / channels of x
    (NHWC float32), float32 arithmetic in the reference's order."""
    n, h, w, c = x.shape
    oh, ow = h + 2 * pad - 2, w + 2 * pad - 2
    th, tw = (oh + 1) // 2, (ow + 1) // 2
    lo = np.full(16, np.inf, np.float32)
    hi = np.full(16, -np.inf, np.float32)
    for i0 in range(0, n, chunk):
        xb = x[i0:i0 + chunk]
        # zero-padded canvas covering every tile window (extract_tiles, tensor.hpp:141-147)
        ph, pw = 2 * th + 2, 2 * tw + 2
        cv = np.zeros((xb.shape[0], ph, pw, c), np.float32)
        cv[:, pad:pad + h, pad:pad + w] = xb
        d = [[cv[:, a:a + 2 * th:2, b:b + 2 * tw:2] for b in range(4)] for a in range(4)]
        # column pass t = B^T d (rows combined per column), then rows
        t = [[None] * 4 for _ in range(4)]
        for b in range(4):
            t[0][b] = d[0][b] - d[2][b]
            t[1][b] = d[1][b] + d[2][b]
            t[2][b] = d[2][b] - d[1][b]
            t[3][b] = d[1][b] - d[3][b]
        for a in range(4):
            v = (t[a][0] - t[a][2], t[a][1] + t[a][2], t[a][2] - t[a][1], t[a][1] - t[a][3])
            for b in range(4):
                p = 4 * a + b
                lo[p] = min(lo[p], v[b].min())
                hi[p] = max(hi[p], v[b].max())
    return lo, hi


@pytest.mark.parametrize("n,c,k,h", LARGE, ids=lambda v: str(v))
def test_config5_extremes(n, c, k, h):
    lo = Oracle()
    rng = np.random.default_rng(n * 7 + c + h)
    x = rng.uniform(-1, 1, size=(n, h, h, c)).astype(np.float32)
    w = (rng.uniform(-1, 1, size=(k, 3, 3, c)) * np.sqrt(2.0 / (9 * c))).astype(np.float32)
    cfg = lance.LanceConfig(8, 8, lance.Granularity.PerPosition, lance.LanceMode.Gemm)
    conv = lance.LanceConv(lance.ConvSpec(n, c, h, h, k, 1), cfg)
    conv.set_filters(torch.from_numpy(w).cuda())
    y = conv.forward(torch.from_numpy(x).cuda())
    conv.sync()
    pa, _ = conv.params()
    arr = lance.params_array(pa)

    # 1. whole-batch fit vs exact host recomputation
    vlo, vhi = v_ranges(x, 1)
    for p in range(16):
        ref = lo.fit_params(np.array([vlo[p], vhi[p]], np.float32), 8)
        got = (pa[p].t_min, pa[p].t_max, pa[p].scale)
        assert np.float32(got[0]) == np.float32(ref.t_min) and np.float32(got[1]) == np.float32(ref.t_max)
        assert np.float32(got[2]).view(np.uint32) == np.float32(ref.scale).view(np.uint32), p

    # 2. output slices vs the oracle with the batch's params
    yh = y.cpu().numpy()
    assert np.isfinite(yh).all()
    s1 = Spec(1, c, h, h, k, 1)
    for img in sorted({0, n // 2, n - 1}):
        ref = lo.lance_gemm(s1, x[img:img + 1], w, in_params=arr)
        bad = int(np.sum(ref.view(np.uint32) != yh[img:img + 1].view(np.uint32)))
        assert bad == 0, f"image {img}: {bad} of {ref.size} outputs differ"
    conv.close()
