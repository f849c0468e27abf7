"""One-screen summary of a bench.py JSON line."""
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(f"value {d['value']:.0f} images/s  ms/step {d['ms_per_step']:.3f}  clocks {d.get('clocks')}")
if d.get("e2e"):
    print("e2e", round(d["e2e"]["value"]), d["e2e"]["unit"])
for k, v in d["roofline"]["stages"].items():
    print(f"  {k:24s} {v['ms_per_step']*1e3:8.1f} us/step  {v['achieved_gbs']:7.0f} GB/s  {100*v['frac_hbm']:5.1f}% HBM")
g = d["roofline"].get("gemm_stage_int8", {})
print("  gemm int8", g)
for l in d["roofline"]["per_layer"]:
    print("  ", l["c"], l["k"], l["h"], l["us_per_forward"])
