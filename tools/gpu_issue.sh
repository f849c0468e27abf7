#!/bin/bash
set -u
OUT=gpurun_out/${1:-issue}
mkdir -p $OUT
for il in 1 2 4 8 1; do
  LANCE_LIB_PATH=scratch/ab_prof/liblance_b200.so LANCE_GEMM_ISSUE_LANES=$il timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > $OUT/il$il.json 2>> $OUT/err.log
  python3 -c "
import json; d=json.load(open('$OUT/il$il.json')); pl=d['roofline']['per_layer']
print('issue_lanes $il', round(d['value']), round(d['ms_per_step'],4), d['parity']['bitexact'], [pl[i]['us_per_forward'][2] for i in (0,4,7,10)])"
done
