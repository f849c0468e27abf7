#!/bin/bash
# Quick GPU iteration: build, parity tests, short bench (no CPU baseline / e2e).
#   gpurun --timeout 900 -- bash tools/gpu_quick.sh <tag> [bench args]
set -u
TAG=${1:-quick}; shift
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || echo "build failed" >> $OUT/build.log
timeout 400 python -m pytest tests -m gpu -x -q --timeout 120 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e "$@" > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
python tools/bench_summary.py $OUT/bench.json > $OUT/summary.txt 2>&1
echo done
