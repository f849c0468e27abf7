"""Top SASS instructions by warp-stall samples from `ncu --page source --csv --print-source sass`."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = rows[2:]
i_src, i_s = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
stall_cols = [k for k, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
tot = sum(float(r[i_s] or 0) for r in data)
print(f"total samples {tot:.0f}")
top = sorted(range(len(data)), key=lambda k: -float(data[k][i_s] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]
for k in sorted(top):
    r = data[k]
    s = float(r[i_s] or 0)
    reasons = sorted(((float(r[c] or 0), h[c][6:]) for c in stall_cols), reverse=True)[:2]
    print(f"{k:5d} {100*s/tot:5.1f}% {r[i_src][:60]:60s} {reasons}")
