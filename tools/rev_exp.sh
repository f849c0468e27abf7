#!/bin/bash
set -u
TAG=$1; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python -m pytest tests -m gpu -x -q --timeout 120 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
for cfg in "LANCE_K1_REVERSE=0" "LANCE_K1_REVERSE=1"; do
  echo "== $cfg" >> $OUT/exp.txt
  env $cfg timeout 120 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > $OUT/b.json 2>> $OUT/exp.err
  python tools/bench_summary.py $OUT/b.json >> $OUT/exp.txt
done
echo done
