"""Condense ncu reports into the numbers the roofline needs (committed under profiles/)."""
import csv, subprocess, sys, io, re, collections

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size"]

def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2]

def stalls(h, v):
    items = [(n.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), float(v[i] or 0))
             for i, n in enumerate(h) if n.startswith("smsp__average_warps_issue_stalled") and n.endswith("per_issue_active.ratio")]
    return sorted(items, key=lambda t: -t[1])[:6]

for rep in sys.argv[1:]:
    h, u, v = raw(rep)
    name = v[h.index("Kernel Name")] if "Kernel Name" in h else rep
    print(f"== {rep}\n   kernel: {name[:110]}")
    for k in KEYS:
        if k in h:
            i = h.index(k)
            print(f"   {k:78s} {v[i]:>16s} {u[i]}")
    print("   top stalls (warps per issue):", ", ".join(f"{n} {x:.2f}" for n, x in stalls(h, v)))
