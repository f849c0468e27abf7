#!/bin/bash
# ncu --set full of one kernel on one bench layer, exported as the raw page and
# the per-SASS-line source page (instructions executed, stall samples).
#   gpurun -- bash tools/prof_src.sh <tag> <kernel-regex> <layer> [skip]
set -u
TAG=$1; K=$2; L=$3; SKIP=${4:-3}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s $SKIP -c 1 \
  -o $OUT/rep_L$L python bench.py --layers $L --steps 1 --warmup 3 --no-cpu --no-e2e --no-verify ${BENCH_ARGS:-} \
  > $OUT/ncu_L$L.log 2>&1
ncu -i $OUT/rep_L$L.ncu-rep --page raw --csv > $OUT/raw_L$L.csv 2>/dev/null
ncu -i $OUT/rep_L$L.ncu-rep --page source --csv --print-source sass > $OUT/src_L$L.csv 2>/dev/null
tot=$(du -sm $OUT | cut -f1); if [ $tot -gt 50 ]; then rm -f $OUT/rep_L$L.ncu-rep; fi
du -sh $OUT/*
