#!/bin/bash
# round-2 re-entry check: full GPU suite, smoke, N=1 bench line, launch list.
set -u
OUT=gpurun_out/${1:-r2c}
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q --durations 10 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-verify > $OUT/ncu_launch.log 2>&1
tail -3 $OUT/pytest_gpu.log; tail -2 $OUT/smoke.log; head -c 1500 $OUT/bench.json; echo; tail -5 $OUT/bench.err
