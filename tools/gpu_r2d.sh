#!/bin/bash
set -u
OUT=gpurun_out/r2d
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -2 $OUT/pytest_gpu.log
bash tools/gpu_ab.sh r2d_ab
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --layout nchw > $OUT/bench_nchw.json 2> $OUT/bench_nchw.err
python3 -c "
import json; d=json.load(open('$OUT/bench_nchw.json')); pl=d['roofline']['per_layer']
print('nchw', round(d['value']), round(d['ms_per_step'],4), d['parity']['bitexact'], [pl[i]['us_per_forward'] for i in (0,4,7,10)])"
