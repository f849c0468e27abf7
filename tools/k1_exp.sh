#!/bin/bash
set -u
TAG=$1; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for cfg in "LANCE_K1_DEPTH=1" "LANCE_K1_DEPTH=2"; do
  echo "== $cfg" >> $OUT/exp.txt
  env $cfg timeout 120 python bench.py --layers 0,4,7,10 --steps 5 --warmup 3 --no-cpu --no-e2e > $OUT/b.json 2>> $OUT/exp.err
  python -c "
import json; d=json.load(open('$OUT/b.json'))
for l in d['roofline']['per_layer']: print('  ', l['c'], l['h'], l['us_per_forward'])" >> $OUT/exp.txt
done
LANCE_K1_DEPTH=2 timeout 300 python -m pytest tests -m gpu -x -q --timeout 120 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
echo done
