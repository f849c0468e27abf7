#!/bin/bash
# Per-layer stage times for several library builds: tools/ab_libs.sh TAG lib1 lib2 ...
set -u
TAG=$1; shift
OUT=gpurun_out/$TAG
mkdir -p $OUT
for rep in 1 2; do
for lib in "$@"; do
  echo "== $lib" >> $OUT/exp.txt
  env LANCE_LIB_PATH=$lib timeout 120 python bench.py --layers ${LAYERS:-0,4,7,10} --steps 5 --warmup 3 --no-cpu --no-e2e ${BENCH_ARGS:-} > $OUT/b.json 2>> $OUT/exp.err
  python -c "
import json; d=json.load(open('$OUT/b.json'))
for l in d['roofline']['per_layer']: print('  ', l['c'], l['h'], l['us_per_forward'])" >> $OUT/exp.txt
done
done
echo done
