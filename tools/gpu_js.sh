#!/bin/bash
set -u
OUT=gpurun_out/${1:-js}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_jsplit.py -x -q > $OUT/pytest_js.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_js.log
tail -3 $OUT/pytest_js.log
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
for js in 1 0; do
  for b in 256 64 32; do
    LANCE_LIB_PATH=scratch/ab_prof/liblance_b200.so LANCE_GEMM_JSPLIT=$js timeout 600 python bench.py --batch $b --steps 20 --warmup 5 --no-cpu --no-e2e > $OUT/js${js}_b$b.json 2>> $OUT/err.log
    python3 -c "
import json; d=json.load(open('$OUT/js${js}_b$b.json')); pl=d['roofline']['per_layer']
print('js $js batch $b', round(d['value']), round(d['ms_per_step'],4), d['parity']['bitexact'], [pl[i]['us_per_forward'][2] for i in (0,4,7,10)])"
  done
  for w in vgg stack; do
    extra=""; [ $w = stack ] && extra="--stack"
    LANCE_LIB_PATH=scratch/ab_prof/liblance_b200.so LANCE_GEMM_JSPLIT=$js timeout 600 python bench.py --workload vgg16_cifar $extra --steps 20 --warmup 5 --no-cpu --no-e2e > $OUT/js${js}_$w.json 2>> $OUT/err.log
    python3 -c "
import json; d=json.load(open('$OUT/js${js}_$w.json')); print('js $js $w', round(d['value']), round(d['ms_per_step'],4), (d.get('parity') or {}).get('bitexact'))"
  done
done
tail -3 $OUT/err.log
