import sys
import numpy as np
a = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(2, 4, 4096).astype(np.int64)
for mode in range(2):
    t = a[mode]
    n = [int(np.count_nonzero(t[i])) for i in range(4)]
    if not n[0]:
        continue
    t0 = t[0][0]
    iss, seen, done, ldr = (t[i][:n[i]] - t0 for i in range(4))
    print(f"== {'K0 range' if mode == 0 else 'K1 quant'}: events {n}")
    m = min(len(iss), len(seen))
    print("  row latency issue->seen: median %d p10 %d p90 %d" % (np.median(seen[:m] - iss[:m]), np.percentile(seen[:m]-iss[:m], 10), np.percentile(seen[:m]-iss[:m], 90)))
    print("  compute done interval: median %d" % np.median(np.diff(done)))
    print("  row issue interval: median %d" % np.median(np.diff(iss)))
    print("  issued :", iss[:24])
    print("  seen   :", seen[:24])
    print("  done   :", done[:12])
    print("  ldr    :", ldr[:12])
