import numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_2003_08646_b200 as lance
from oracle import Oracle, Spec
from tests.golden_cases import make_inputs
o = Oracle()
for spec in [Spec(1, 256, 14, 14, 256, 1), Spec(1, 160, 8, 8, 32, 1), Spec(1, 128, 8, 8, 32, 1), Spec(1, 256, 8, 8, 32, 1)]:
    x, w = make_inputs(o.uniform, spec, "uniform", 42)
    y, ref = o.lance_gemm(spec, x, w, dump=True)
    conv = lance.LanceConv(lance.ConvSpec(spec.n, spec.c, spec.h, spec.w, spec.k, spec.pad),
                           lance.LanceConfig(8, 8, lance.Granularity.PerPosition, lance.LanceMode.Gemm))
    acc = torch.empty((16, spec.rows, spec.k), dtype=torch.int32, device='cuda')
    conv.set_acc_dump(acc)
    conv.set_filters(torch.from_numpy(w).cuda())
    g = conv.forward(torch.from_numpy(x).cuda()); conv.sync()
    g = g.cpu().numpy()
    bad = g.view(np.uint32) != y.view(np.uint32)
    print(spec, "acc ok", np.array_equal(acc.cpu().numpy(), ref["acc"]), "bad y", bad.sum(), "of", bad.size)
    if bad.any():
        idx = np.argwhere(bad)
        print(" filters with errors:", np.unique(idx[:, 3])[:40])
        print(" rows (oy) with errors:", np.unique(idx[:, 1])[:20], "cols", np.unique(idx[:, 2])[:20])
        i = tuple(idx[0]); print(" first", i, g[i], y[i])
