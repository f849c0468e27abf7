#!/bin/bash
set -u
OUT=gpurun_out/${1:-rs}
mkdir -p $OUT
for r in 1 0 1 0; do
  LANCE_LIB_PATH=scratch/ab_prof/liblance_b200.so LANCE_RS_GEMM=$r timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > $OUT/rs$r.json 2>> $OUT/err.log
  python3 -c "
import json; d=json.load(open('$OUT/rs$r.json')); pl=d['roofline']['per_layer']
print('rs_gemm $r', round(d['value']), round(d['ms_per_step'],4), d['parity']['bitexact'], [pl[i]['us_per_forward'] for i in (0,4)])"
done
