"""Run one layer with a trace-enabled library (tools/band_trace.sh) and dump the band kernels'
CTA-0 clock64 stamps: [mode K0/K1][slot: 0 row issued, 1 row seen by warp 0, 2 compute done,
3 loader saw stage_full][index].  Scratch / profiling only."""
import ctypes as ct, sys, torch
import numpy as np
sys.path.insert(0, '.')
import paper_2003_08646_b200 as lance
from paper_2003_08646_b200 import _lib
c, h, n, out = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
spec = lance.ConvSpec(n, c, h, h, c, 1)
cfg = lance.LanceConfig(8, 8, lance.Granularity.PerPosition, lance.LanceMode.Gemm)
conv = lance.LanceConv(spec, cfg)
conv.set_filters(torch.rand(c, 3, 3, c, device='cuda') * 2 - 1)
x = torch.rand(n, h, h, c, device='cuda') * 2 - 1
for _ in range(3):
    conv.forward(x)
conv.sync()
buf = np.zeros(8 * 4096, np.uint64)
lib = ct.CDLL(_lib.LIB_PATH)
rc = lib.lance_debug_band_trace(buf.ctypes.data_as(ct.c_void_p), ct.c_size_t(buf.nbytes))
print("rc", rc)
buf.tofile(out)
