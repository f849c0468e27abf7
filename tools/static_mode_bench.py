#!/usr/bin/env python3
"""Per-stage times of the dynamic (range pass + fit) and static-params
(caller QuantParams: the full-batch-parity multi-GPU mode of shard.py) forwards
on one layer shape."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2003_08646_b200 as lance  # noqa: E402

for c, h in ((64, 56), (256, 14)):
    spec = lance.ConvSpec(256, c, h, h, c, 1)
    cfg = lance.LanceConfig(8, 8, lance.Granularity.PerPosition, lance.LanceMode.Gemm)
    conv = lance.LanceConv(spec, cfg)
    x = torch.rand((256, h, h, c), device="cuda") * 2 - 1
    conv.set_filters(torch.rand((c, 3, 3, c), device="cuda") * 2 - 1)
    y = conv.forward(x)
    conv.sync()
    params, _ = conv.params()
    out = {}
    for mode, prm in (("dynamic", None), ("static", params)):
        for _ in range(3):
            conv.forward(x, y, params=prm)
        conv.sync()
        conv.stage_timing(True)
        for _ in range(10):
            conv.forward(x, y, params=prm)
        ms, n = conv.read_stage_times()
        conv.stage_timing(False)
        out[mode] = [round(m / n * 1e3, 1) for m in ms]
    print(json.dumps({"c": c, "h": h, "us_K0_K1_GEMM": out}))
