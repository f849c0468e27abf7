#!/bin/bash
# PDL A/B: release build (PDL on) bench + GPU tests, then a LANCE_PROFILING
# build with LANCE_PDL=0/1.
set -u
OUT=gpurun_out/${1:-pdl}
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > $OUT/bench_on.json 2> $OUT/bench_on.err
LANCE_PROFILING=1 python -m paper_2003_08646_b200.build --force > /dev/null 2>&1
for v in 0 1 0 1; do
  LANCE_PDL=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-verify > $OUT/bench_pdl$v.json 2>> $OUT/bench_ab.err
  python3 -c "import json; d=json.load(open('$OUT/bench_pdl$v.json')); print('PDL=$v', round(d['value']), round(d['ms_per_step'],4))"
done
tail -2 $OUT/pytest_gpu.log
python3 -c "import json; d=json.load(open('$OUT/bench_on.json')); print('release', round(d['value']), d['ms_per_step'], d.get('parity'))"
