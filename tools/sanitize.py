#!/usr/bin/env python3
"""Small driver for compute-sanitizer (memcheck / racecheck / synccheck) over
every kernel family of the library: F(2x2) K0/K1 (fast strip, generic, small-C,
static params), the NCHW staging transpose, the tcgen05 GEMM at BN = 16/32/64
with and without the acc dump and resident B, its fused max-pool and j-split
modes, F(4x4) F0/F1/F3, and the max-pool kernel.  Run under gpurun:

    compute-sanitizer --tool memcheck  python tools/sanitize.py [--big]
    compute-sanitizer --tool racecheck python tools/sanitize.py
    compute-sanitizer --tool synccheck python tools/sanitize.py

--big adds the R512 bench layer at N = 256 (256 GEMM tiles over 148 CTAs,
i.e. several tiles per persistent CTA) -- memcheck only, racecheck is too slow.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2003_08646_b200 as lance  # noqa: E402

CFG = lance.LanceConfig(8, 8, lance.Granularity.PerPosition, lance.LanceMode.Gemm)


def run(n, c, h, k, pad=1, tile_m=2, acc=False, static=False, bias=False, layout="nhwc", pool=False):
    spec = lance.ConvSpec(n, c, h, h, k, pad)
    conv = lance.LanceConv(spec, CFG, tile_m=tile_m, layout=layout)
    g = torch.Generator(device="cpu").manual_seed(n * 131 + c * 7 + h + k)
    x = torch.randn((n, c, h, h) if layout == "nchw" else (n, h, h, c), generator=g).cuda()
    w = torch.randn((k, 3, 3, c), generator=g).cuda()
    conv.set_filters(w)
    if bias or pool:
        conv.set_epilogue(torch.randn(k, generator=g).cuda(), relu=True, pool=pool)
    if acc:
        conv.set_acc_dump(torch.empty((conv.positions, conv.rows, k), dtype=torch.int32, device="cuda"))
    y = conv.forward(x)
    conv.sync()
    if static:
        pa, _ = conv.params()
        y2 = conv.forward(x, params=pa)
        conv.sync()
        assert torch.equal(y, y2)
    conv.close()
    torch.cuda.synchronize()
    return float(y.abs().sum())


def main():
    cases = [
        dict(n=2, c=64, h=17, k=64),                 # fast K0/K1, GEMM BN=64->32, row sums in GEMM
        dict(n=1, c=128, h=14, k=64, acc=True),      # BK=128, row sums in K1, acc dump
        dict(n=1, c=96, h=11, k=24, pad=0),          # generic K1, BN=32
        dict(n=3, c=3, h=13, k=20, static=True),     # small-C kernels, static params
        dict(n=1, c=64, h=9, k=16, bias=True),       # BN=16, bias+ReLU epilogue
        dict(n=1, c=64, h=16, k=32, tile_m=4),       # F(4x4)
        dict(n=1, c=128, h=12, k=48, tile_m=4, acc=True),
        dict(n=2, c=40, h=13, k=24, layout="nchw"),  # NCHW staging transpose (scalar path)
        dict(n=2, c=64, h=16, k=64, layout="nchw"),  # NCHW (128-bit path)
        dict(n=2, c=64, h=15, k=96, pool=True),      # fused 2x2 max-pool epilogue, odd map
        dict(n=4, c=256, h=7, k=128),                # GEMM j-split (4 CTAs per tile)
        dict(n=2, c=256, h=9, k=100, acc=True),      # j-split, partial filter tile, acc dump
    ]
    if "--big" in sys.argv:
        cases += [dict(n=256, c=512, h=7, k=512), dict(n=32, c=64, h=56, k=64, tile_m=4),
                  dict(n=32, c=512, h=7, k=512)]  # j-split at the 8-GPU per-rank batch
    for cs in cases:
        print(cs, run(**cs), flush=True)
    a = torch.randn(2, 8, 8, 16, device="cuda")
    b = torch.empty(2, 4, 4, 16, device="cuda")
    lance.api._check(lance._lib.lib().lance_maxpool2x2_nhwc(
        a.data_ptr(), b.data_ptr(), 2, 8, 8, 16, torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    print("sanitize driver done")


if __name__ == "__main__":
    main()
