"""Summarise a GEMM CTA-0 trace (tools/trace.sh): per-tile / per-j-group
timeline of the producer, the MMA issuer and epilogue warp 0, in SM cycles."""
import sys

import numpy as np

SL = 100000
names = {0: "prod_issue", 1: "mma_full", 2: "mma_commit", 7: "mma_grp_start", 6: "epi_rs_ready",
         3: "epi_acc_full", 4: "epi_acc_release", 5: "epi_grp_done"}
t = np.fromfile(sys.argv[1], dtype=np.uint64).astype(np.int64).reshape(5, SL) if False else None
raw = np.fromfile(sys.argv[1], dtype=np.uint64).astype(np.int64)
slots = {k: raw[k * SL:(k + 1) * SL] for k in range(8) if (k + 1) * SL <= raw.size}
t0 = min(v[v > 0].min() for v in slots.values() if (v > 0).any())
ser = {k: (v[v > 0] - t0) for k, v in slots.items()}
for k in sorted(ser):
    v = ser[k]
    if v.size:
        print(f"{names.get(k, k):16s} n={v.size:5d} first={v[0]:8d} last={v[-1]:8d} mean_gap={np.diff(v).mean() if v.size > 1 else 0:8.1f}")
stages_per_grp = int(sys.argv[2]) if len(sys.argv) > 2 else 0
g0 = ser.get(7, np.array([]))
for i in range(min(len(g0), 12)):
    row = [f"{names[k][:12]}={ser[k][i]:7d}" for k in (7, 6, 3, 4, 5) if k in ser and i < ser[k].size]
    print(f"grp {i:2d}: " + " ".join(row))
if stages_per_grp:
    f, c = ser[1], ser[2]
    n = min(f.size, c.size)
    print("MMA busy per stage (commit - full):", np.mean(c[:n] - f[:n]).round(1),
          " MMA wait per stage (full_k - commit_{k-1}):", np.mean(f[1:n] - c[:n - 1]).round(1))
    p = ser[0]
    print("producer issue gap mean:", np.diff(p).mean().round(1), " producer lead over MMA full (stages):",
          np.mean([np.searchsorted(p, x) for x in f[:n]] - np.arange(n)).round(2))
