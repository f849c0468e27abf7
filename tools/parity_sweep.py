#!/usr/bin/env python3
"""Randomised GPU parity sweep (one-off confidence check beyond tests/):
random shapes / seeds / paddings / C in {64, 128, 192, 256} (fast strip and
staged paths) and odd C, F(2x2) and F(4x4), each compared bitwise with the
oracle on y and the u8 codes.  Prints one line per case and a summary."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2003_08646_b200 as lance  # noqa: E402
from oracle import Oracle, Spec  # noqa: E402
from tests.golden.make_golden import make_inputs  # noqa: E402

o = Oracle()
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 2026)
cfg = lance.LanceConfig(8, 8, lance.Granularity.PerPosition, lance.LanceMode.Gemm)
bad = 0
n_cases = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for i in range(n_cases):
    c = int(rng.choice([64, 128, 192, 256, 96, 40, 7]))
    k = int(rng.choice([16, 24, 64, 80, 128, 192]))
    h, w = int(rng.integers(5, 23)), int(rng.integers(5, 23))
    n = int(rng.integers(1, 4))
    pad = int(rng.integers(0, 2))
    tm = int(rng.choice([2, 4]))
    spec = Spec(n, c, h, w, k, pad)
    x, wt = make_inputs(o.uniform, spec, str(rng.choice(["relu", "uniform"])), int(rng.integers(1, 1000)))
    conv = lance.LanceConv(lance.ConvSpec(n, c, h, w, k, pad), cfg, tile_m=tm)
    conv.set_filters(torch.from_numpy(wt).cuda())
    y = conv.forward(torch.from_numpy(x).cuda())
    conv.sync()
    got = y.cpu().numpy()
    codes = conv.debug_read("codes_a")
    conv.close()
    ref, d = o.lance_gemm(spec, x, wt, dump=True, tile_m=tm)
    ok = np.array_equal(got.view(np.uint32), ref.view(np.uint32)) and np.array_equal(codes, d["codes_a"])
    bad += 0 if ok else 1
    print(f"{'ok ' if ok else 'BAD'} F({tm}x{tm}) N={n} C={c} H={h} W={w} K={k} pad={pad}", flush=True)
print(f"summary: {n_cases - bad}/{n_cases} bit-exact")
sys.exit(1 if bad else 0)
