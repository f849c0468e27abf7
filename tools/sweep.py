#!/usr/bin/env python3
"""sweep C, K in {64..512}, H in {7..112},
N in {1..1024} through the device API, one JSON row per shape with images/s,
per-stage microseconds and each stage's algorithmic HBM GB/s vs the measured
peak (bench.py's stage_bytes).  Shapes whose batch of activations would not
fit comfortably in HBM are skipped.

    python tools/sweep.py [--tile-m 2] [--quick] > profiles/r01_sweep.jsonl
"""
from __future__ import annotations

import argparse
import itertools
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tile-m", type=int, default=2, choices=(2, 4))
    ap.add_argument("--quick", action="store_true", help="a 24-shape subset")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    import numpy as np
    import torch
    import paper_2003_08646_b200 as lance

    dev = torch.device("cuda", 0)
    hbm, _ = bench.peaks()
    cfg = lance.LanceConfig(8, 8, lance.Granularity.PerPosition, lance.LanceMode.Gemm)
    cs = (64, 128, 256, 512)
    hs = (7, 14, 28, 56, 112)
    ns = (1, 8, 64, 256, 1024)
    shapes = [(c, c, h, n) for c, h, n in itertools.product(cs, hs, ns)]
    shapes += [(c, k, 28, 64) for c, k in itertools.product(cs, cs) if c != k]
    if a.quick:
        shapes = [s for s in shapes if s[3] in (8, 256) and s[2] in (7, 28, 112)]
    for c, k, h, n in shapes:
        xbytes = 4 * n * h * h * c
        if xbytes * 4.5 > 60e9:  # x, y and codes of one layer must fit with margin
            continue
        spec = lance.ConvSpec(n, c, h, h, k, 1)
        x = torch.rand((n, h, h, c), device=dev) * 2 - 1
        w = torch.rand((k, 3, 3, c), device=dev) * 2 - 1
        conv = lance.LanceConv(spec, cfg, tile_m=a.tile_m)
        conv.set_filters(w)
        y = torch.empty((n, h, h, k), device=dev)
        for _ in range(2):
            conv.forward(x, y)
        conv.sync()
        conv.stage_timing(True)
        for _ in range(a.reps):
            conv.forward(x, y)
        ms, nf = conv.read_stage_times()
        conv.stage_timing(False)
        conv.sync()
        us = [m / nf * 1e3 for m in ms]
        tot = sum(us)
        sb = bench.stage_bytes(c, k, h, n, a.tile_m)
        row = {"c": c, "k": k, "h": h, "n": n, "winograd": f"F({a.tile_m}x{a.tile_m},3x3)",
               "us": [round(u, 2) for u in us], "images_per_s": n / (tot * 1e-6),
               "tops_equivalent": 2 * bench.direct_macs(c, k, h, n) / (tot * 1e-6) / 1e12,
               "frac_hbm": [round(b / (u * 1e-6) / 1e9 / hbm, 3) for b, u in zip(sb, us)]}
        print(json.dumps(row), flush=True)
        conv.close()
        del x, w, y
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
