#!/bin/bash
set -u
OUT=gpurun_out/${1:-fused}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_parity.py tests/test_gpu_large.py tests/test_gpu_multi.py -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
tail -3 $OUT/pytest.log
for b in 256 128 64 32; do for f in 0 1; do for rep in 1; do
  LANCE_LIB_PATH=scratch/ab_prof/liblance_b200.so LANCE_FUSED_INPUT=$f timeout 600 python bench.py --batch $b --steps 20 --warmup 5 --no-cpu --no-e2e > $OUT/b${b}_f${f}_$rep.json 2>> $OUT/err.log
  python3 -c "
import json; d=json.load(open('$OUT/b${b}_f${f}_$rep.json')); pl=d['roofline']['per_layer']
print('batch $b fused $f', round(d['value']), round(d['ms_per_step'],4), d['parity']['bitexact'], [pl[i]['us_per_forward'] for i in (0,4,7,10)])"
done; done; done
tail -3 $OUT/err.log
