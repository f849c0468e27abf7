#!/bin/bash
set -u
OUT=gpurun_out/${1:-lanes}
mkdir -p $OUT
for ll in 1 2 4 8 1 4; do
  LANCE_LIB_PATH=scratch/ab_prof/liblance_b200.so LANCE_GEMM_LANES=$ll timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > $OUT/ll${ll}.json 2>> $OUT/err.log
  python3 -c "
import json; d=json.load(open('$OUT/ll$ll.json')); pl=d['roofline']['per_layer']
print('ld_lanes $ll', round(d['value']), round(d['ms_per_step'],4), d['parity']['bitexact'], [pl[i]['us_per_forward'][2] for i in (0,4,7,10)])"
done
