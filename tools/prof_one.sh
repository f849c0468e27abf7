#!/bin/bash
# ncu --set full of one kernel family on given bench layers.
#   gpurun -- bash tools/prof_one.sh <tag> <kernel-regex> <layer> [<layer> ...]
set -u
TAG=$1; K=$2; shift 2
SKIP=${SKIP:-3}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for L in "$@"; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s $SKIP -c 1 \
    -o $OUT/${K}_L$L python bench.py --layers $L --steps 1 --warmup 3 --no-cpu --no-e2e ${BENCH_ARGS:-} \
    > $OUT/ncu_${K}_L$L.log 2>&1
done
echo done
