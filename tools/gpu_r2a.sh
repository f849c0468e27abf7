#!/bin/bash
# Round-2 GPU check: full GPU test suite (incl. the batch-256 bench-shape parity
# tests), compute-sanitizer passes, one bench line.
set -u
OUT=gpurun_out/${1:-r2a}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
for tool in memcheck racecheck synccheck; do
  extra=""; [ $tool = memcheck ] && extra="--big"
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize.py $extra > $OUT/sanitize_$tool.log 2>&1; echo "rc=$?" >> $OUT/sanitize_$tool.log
done
timeout 600 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err
tail -3 $OUT/pytest_gpu.log; tail -2 $OUT/sanitize_*.log; head -c 600 $OUT/bench.json
