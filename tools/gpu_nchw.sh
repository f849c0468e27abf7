#!/bin/bash
set -u
OUT=gpurun_out/${1:-nchw}
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -2 $OUT/pytest_gpu.log
for L in nhwc nchw; do
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --layout $L > $OUT/bench_$L.json 2> $OUT/bench_$L.err
python3 -c "
import json; d=json.load(open('$OUT/bench_$L.json')); pl=d['roofline']['per_layer']
print('$L', round(d['value']), round(d['ms_per_step'],4), d['parity']['bitexact'], [pl[i]['us_per_forward'] for i in (0,4,7,10)])"
done
