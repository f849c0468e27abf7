"""Summarise a GEMM CTA-0 trace: slots 0 producer issued / 1 MMA full-ready / 2 producer slot-free /
3 epilogue acc-full-ready / 4 epilogue release (clock64 cycles)."""
import sys
import numpy as np
a = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(5, 100000).astype(np.int64)
n = [int(np.count_nonzero(a[i])) for i in range(5)]
t0 = min(a[i][a[i] > 0].min() for i in range(5) if n[i])
print("events", n)
prod, full, aempty, afull, rel = (a[i][:n[i]] - t0 for i in range(5))
print("total cycles", max(x.max() for x in (prod, full, aempty, afull, rel) if len(x)))
def d(x): return np.diff(x) if len(x) > 1 else np.array([0])
print("producer issue interval  median %d  mean %.0f" % (np.median(d(prod)), d(prod).mean()))
print("MMA full-ready interval  median %d  mean %.0f" % (np.median(d(full)), d(full).mean()))
m = min(len(prod), len(full))
print("stage latency (issue->ready)  median %d  p90 %d" % (np.median(full[:m] - prod[:m]), np.percentile(full[:m] - prod[:m], 90)))
g = min(len(afull), len(rel), len(aempty))
print("group: epi ready->release median %d; group interval %d" % (np.median(rel[:g] - afull[:g]), np.median(d(afull))))
g2=min(len(prod),len(aempty))
print("producer: slot-free -> issued median %d; issued -> next slot-free median %d" % (np.median(prod[:g2]-aempty[:g2]), np.median(aempty[1:g2]-prod[:g2-1])))
print(" slot_free first 20", aempty[:20])
print(" epi_acc_full   ", afull[:12])
print(" epi_release    ", rel[:12])
print(" prod first 20  ", prod[:20])
print(" full first 20  ", full[:20])
