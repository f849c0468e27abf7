#!/bin/bash
set -u
OUT=gpurun_out/${1:-units}
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
for b in 256 32; do for u in def 1 2; do
  if [ $u = def ]; then env=""; else env="LANCE_GEMM_UNITS=$u"; fi
  env LANCE_LIB_PATH=scratch/ab_prof/liblance_b200.so $env timeout 600 python bench.py --batch $b --steps 20 --warmup 5 --no-cpu --no-e2e > $OUT/b${b}_u$u.json 2>> $OUT/err.log
  python3 -c "
import json; d=json.load(open('$OUT/b${b}_u$u.json')); pl=d['roofline']['per_layer']
print('batch $b units $u', round(d['value']), round(d['ms_per_step'],4), d['parity']['bitexact'], [pl[i]['us_per_forward'] for i in (0,4,7,10)])"
done; done
