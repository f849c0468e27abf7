"""GEMM j-split (small-M layers): a tile's 4 j-groups on 4 CTAs, the last to
finish completing the left fold of A^T m A from the exchanged T0j / T1j.  The
result must be bit-identical to the single-CTA fold and to the oracle
(lance_gemm, engines.hpp:492-536; fold order matrix.hpp:75-84), including the
raw int32 accumulators, bias + ReLU, ragged maps, K not a multiple of 64 and
several tiles per CTA (more units than SMs are never planned, so multi-unit
CTAs come from a small grid).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2003_08646_b200 as lance  # noqa: E402
from oracle import Oracle, Spec  # noqa: E402

pytestmark = pytest.mark.gpu


def cfg():
    return lance.LanceConfig(8, 8, lance.Granularity.PerPosition, lance.LanceMode.Gemm)


@pytest.mark.parametrize("shape", [
    (32, 512, 512, 7, 1),   # R512 at the 8-GPU per-rank batch: 32 tiles -> 128 units
    (4, 256, 100, 9, 1),    # K = 100: 2 filter tiles, the second partial
    (3, 128, 64, 11, 0),    # pad 0, ragged 9x9 output
    (1, 64, 96, 13, 1),     # tiny M
    (128, 512, 512, 4, 1),  # VGG-16-CIFAR 4x4 layer
])
def test_jsplit_matches_oracle(shape):
    n, c, k, h, pad = shape
    lo = Oracle()
    spec = Spec(n, c, h, h, k, pad)
    x, w = lo.layer(spec, 5 + c + k)
    conv = lance.LanceConv(lance.ConvSpec(n, c, h, h, k, pad), cfg())
    conv.set_filters(torch.from_numpy(w).cuda())
    acc = torch.empty((16, spec.rows, k), dtype=torch.int32, device="cuda")
    conv.set_acc_dump(acc)
    y = conv.forward(torch.from_numpy(x).cuda())
    conv.sync()
    ref, d = lo.lance_gemm(spec, x, w, dump=True)
    assert np.array_equal(acc.cpu().numpy(), d["acc"])
    assert np.array_equal(y.cpu().numpy().view(np.uint32), ref.view(np.uint32))
    # again without the dump (the production instantiation), twice: the per-tile
    # tickets reset themselves
    conv.set_acc_dump(None)
    for _ in range(2):
        y2 = conv.forward(torch.from_numpy(x).cuda())
        conv.sync()
        assert np.array_equal(y2.cpu().numpy().view(np.uint32), ref.view(np.uint32))
    conv.close()


def test_jsplit_bias_relu():
    lo = Oracle()
    spec = Spec(8, 256, 7, 7, 192, 1)
    x, w = lo.layer(spec, 77)
    b = (lo.uniform(4, 192) * np.float32(0.3)).astype(np.float32)
    conv = lance.LanceConv(lance.ConvSpec(8, 256, 7, 7, 192, 1), cfg())
    conv.set_filters(torch.from_numpy(w).cuda())
    conv.set_epilogue(torch.from_numpy(b).cuda(), relu=True)
    y = conv.forward(torch.from_numpy(x).cuda())
    conv.sync()
    ref = np.maximum(lo.lance_gemm(spec, x, w) + b, np.float32(0)) + np.float32(0)
    assert np.array_equal(y.cpu().numpy().view(np.uint32), ref.astype(np.float32).view(np.uint32))
    conv.close()
