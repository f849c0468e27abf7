#!/bin/bash
set -u
TAG=$1
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for rep in 1 2; do
for lib in scratch/ab_old/liblance_b200.so paper_2003_08646_b200/_build/liblance_b200.so; do
  for cfg in "" "LANCE_GEMM_EXP=3"; do
    echo "== $lib $cfg" >> $OUT/exp.txt
    env LANCE_LIB_PATH=$lib $cfg timeout 120 python bench.py --layers 0,4,7,10 --steps 5 --warmup 3 --no-cpu --no-e2e > $OUT/b.json 2>> $OUT/exp.err
    python -c "
import json; d=json.load(open('$OUT/b.json'))
for l in d['roofline']['per_layer']: print('  ', l['c'], l['h'], l['us_per_forward'])" >> $OUT/exp.txt
  done
done
done
echo done
