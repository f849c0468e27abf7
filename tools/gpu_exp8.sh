#!/bin/bash
set -u
OUT=gpurun_out/${1:-exp8}
mkdir -p $OUT
for e in 0 8 1; do
  LANCE_LIB_PATH=scratch/ab_exp8/liblance_b200.so LANCE_GEMM_EXP=$e timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-verify > $OUT/e$e.json 2>> $OUT/err.log
  python3 -c "
import json; d=json.load(open('$OUT/e$e.json')); pl=d['roofline']['per_layer']
print('exp $e', round(d['ms_per_step'],4), [pl[i]['us_per_forward'][2] for i in (0,4,7,10)])"
done
