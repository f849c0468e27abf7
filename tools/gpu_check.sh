#!/bin/bash
# One gpurun call: GPU parity tests, a short bench, the ncu launch list.
#   gpurun --timeout 1500 -- bash tools/gpu_check.sh [tag]
set -u
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || echo "build failed" >> $OUT/build.log
timeout 600 python -m pytest tests -m gpu -x -q --timeout 120 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 400 python bench.py --steps 10 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 117 -c 39 --csv \
  --log-file $OUT/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > $OUT/ncu_launch.log 2>&1
echo done
