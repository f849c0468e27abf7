"""Layer-stack driver (paper_2003_08646_b200/stack.py) on the GPU: chained
LANCE convs with the fused bias + ReLU epilogue and 2x2 max-pools, eager and as
a replayed CUDA graph, bitwise against the oracle's lance_gemm chained on the
host with relu(y + b) and the pool applied in numpy."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2003_08646_b200 as lance  # noqa: E402
from paper_2003_08646_b200.stack import LanceStack  # noqa: E402
from oracle import Oracle, Spec  # noqa: E402

pytestmark = pytest.mark.gpu

MINI_VGG = [("conv", 3, 16), ("conv", 16, 16), ("pool",), ("conv", 16, 32), ("conv", 32, 24),
            ("pool",), ("conv", 24, 16)]


def host_chain(lo, layers, x, weights, biases, tile_m):
    cur = x
    outs = []
    wi = 0
    for layer in layers:
        if layer[0] == "conv":
            n, h, w, c = cur.shape
            spec = Spec(n, c, h, w, layer[2], 1)
            y = lo.lance_gemm(spec, cur, weights[wi], tile_m=tile_m)
            y = np.maximum(y + biases[wi], np.float32(0.0)) + np.float32(0.0)
            wi += 1
        else:
            n, h, w, c = cur.shape
            v = cur[:, : h // 2 * 2, : w // 2 * 2].reshape(n, h // 2, 2, w // 2, 2, c)
            y = v.max(axis=(2, 4))
        cur = y.astype(np.float32)
        outs.append(cur)
    return outs


@pytest.mark.parametrize("tile_m,fuse", [(2, True), (2, False), (4, False)])
def test_stack_eager_and_graph_bitexact(tile_m, fuse):
    lo = Oracle()
    n, h = 2, 16
    x = np.maximum(lo.uniform(5, n * h * h * 3).reshape(n, h, h, 3), 0).astype(np.float32)
    weights, biases = [], []
    for i, layer in enumerate(l for l in MINI_VGG if l[0] == "conv"):
        _, c, k = layer
        weights.append((lo.uniform(100 + i, k * 9 * c) * np.float32(0.3)).reshape(k, 3, 3, c))
        biases.append((lo.uniform(200 + i, k) * np.float32(0.1)).astype(np.float32))
    cfg = lance.LanceConfig(8, 8, lance.Granularity.PerPosition, lance.LanceMode.Gemm)
    stack = LanceStack(MINI_VGG, n, h, h, cfg, tile_m=tile_m, fuse_pool=fuse)
    assert stack.launches_per_forward() == 5 * 3 + (0 if fuse else 2)
    wd = [torch.from_numpy(w).cuda() for w in weights]
    bd = [torch.from_numpy(b).cuda() for b in biases]
    stack.set_weights(wd, bd)
    xd = torch.from_numpy(x).cuda()
    expect = host_chain(lo, MINI_VGG, x, weights, biases, tile_m)

    y = stack.forward(xd)
    stack.sync()
    for i, (st, e) in enumerate(zip(stack.stages, expect)):
        if i + 1 < len(stack.stages) and stack.stages[i + 1].fused:
            e = expect[i + 1]  # the conv's epilogue wrote the pooled map
        assert np.array_equal(st.out.cpu().numpy().view(np.uint32), e.view(np.uint32)), st.kind
    assert tuple(y.shape) == expect[-1].shape

    # CUDA graph: capture once, replay on a new batch.
    yg = stack.capture(xd)
    torch.cuda.synchronize()
    assert np.array_equal(yg.cpu().numpy().view(np.uint32), expect[-1].view(np.uint32))
    x2 = np.maximum(lo.uniform(6, n * h * h * 3).reshape(n, h, h, 3), 0).astype(np.float32)
    yg = stack.replay(torch.from_numpy(x2).cuda())
    torch.cuda.synchronize()
    expect2 = host_chain(lo, MINI_VGG, x2, weights, biases, tile_m)
    assert np.array_equal(yg.cpu().numpy().view(np.uint32), expect2[-1].view(np.uint32))
    stack.close()


def test_maxpool_odd_dims():
    n, h, w, c = 2, 7, 5, 6
    x = np.random.default_rng(0).standard_normal((n, h, w, c)).astype(np.float32)
    y = torch.empty((n, h // 2, w // 2, c), device="cuda")
    from paper_2003_08646_b200 import _lib
    import ctypes as ct
    xd = torch.from_numpy(x).cuda()
    assert _lib.lib().lance_maxpool2x2_nhwc(ct.c_void_p(xd.data_ptr()), ct.c_void_p(y.data_ptr()),
                                            n, h, w, c, None) == 0
    torch.cuda.synchronize()
    ref = x[:, :6, :4].reshape(n, 3, 2, 2, 2, c).max(axis=(2, 4))
    assert np.array_equal(y.cpu().numpy(), ref)


@pytest.mark.parametrize("shape", [(2, 16, 13, 11, 24, 1), (1, 32, 16, 16, 22, 1), (3, 64, 9, 12, 64, 0),
                                   (4, 128, 28, 28, 128, 1)])
def test_fused_pool_epilogue(shape):
    """lance_plan_set_epilogue_pool: maxpool2x2(relu(lance_gemm(x, w) + b)) in
    the GEMM epilogue, odd maps (floor pooling), K % 4 != 0, pad 0."""
    lo = Oracle()
    n, c, h, w, k, pad = shape
    spec = Spec(n, c, h, w, k, pad)
    x, wt = lo.layer(spec, 11 + c)
    b = (lo.uniform(3, k) * np.float32(0.2)).astype(np.float32)
    cfg = lance.LanceConfig(8, 8, lance.Granularity.PerPosition, lance.LanceMode.Gemm)
    conv = lance.LanceConv(lance.ConvSpec(n, c, h, w, k, pad), cfg)
    conv.set_filters(torch.from_numpy(wt).cuda())
    bd = torch.from_numpy(b).cuda()
    conv.set_epilogue(bd, relu=True, pool=True)
    y = conv.forward(torch.from_numpy(x).cuda())
    conv.sync()
    full = np.maximum(lo.lance_gemm(spec, x, wt) + b, np.float32(0.0)) + np.float32(0.0)
    oh, ow = full.shape[1], full.shape[2]
    ref = full[:, : oh // 2 * 2, : ow // 2 * 2].reshape(n, oh // 2, 2, ow // 2, 2, k).max(axis=(2, 4))
    assert tuple(y.shape) == ref.shape
    assert np.array_equal(y.cpu().numpy().view(np.uint32), ref.astype(np.float32).view(np.uint32))
    conv.close()
