#!/bin/bash
set -u
TAG=$1
OUT=gpurun_out/$TAG
mkdir -p $OUT
for JM in 0 1; do
  LANCE_JMAJOR=$JM python -c "from paper_2003_08646_b200 import build; build.build(force=True)" > $OUT/build$JM.log 2>&1
  for cfg in "" "LANCE_GEMM_EXP=3" "LANCE_GEMM_PF=0" "LANCE_GEMM_BN=64"; do
    echo "== JMAJOR=$JM $cfg" >> $OUT/exp.txt
    env $cfg timeout 120 python bench.py --layers 0,4,7,10 --steps 5 --warmup 3 --no-cpu --no-e2e > $OUT/b.json 2>> $OUT/exp.err
    python -c "
import json; d=json.load(open('$OUT/b.json'))
for l in d['roofline']['per_layer']: print('  ', l['c'], l['h'], l['us_per_forward'])" >> $OUT/exp.txt
  done
done
timeout 300 python -m pytest tests -m gpu -x -q --timeout 120 > $OUT/pytest_jm1.log 2>&1
LANCE_JMAJOR=0 python -c "from paper_2003_08646_b200 import build; build.build(force=True)" > /dev/null 2>&1
timeout 300 python -m pytest tests -m gpu -x -q --timeout 120 > $OUT/pytest_jm0.log 2>&1
echo done
