"""Run one layer a few times with LANCE_GEMM_TRACE set; the plan dumps CTA-0 timestamps on close."""
import sys, torch
sys.path.insert(0, '.')
import paper_2003_08646_b200 as lance
c, h, n = map(int, sys.argv[1:4])
spec = lance.ConvSpec(n, c, h, h, c, 1)
cfg = lance.LanceConfig(8, 8, lance.Granularity.PerPosition, lance.LanceMode.Gemm)
conv = lance.LanceConv(spec, cfg)
conv.set_filters(torch.rand(c, 3, 3, c, device='cuda') * 2 - 1)
x = torch.rand(n, h, h, c, device='cuda') * 2 - 1
for _ in range(3):
    conv.forward(x)
conv.sync()
conv.close()
print("ok")
