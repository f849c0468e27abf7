#!/bin/bash
set -u
OUT=gpurun_out/${1:-tests}
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 1500 python tools/parity_sweep.py 777 200 > $OUT/parity_sweep.log 2>&1; echo "rc=$?" >> $OUT/parity_sweep.log
tail -2 $OUT/pytest_gpu.log; tail -2 $OUT/parity_sweep.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > $OUT/bench.json 2>> $OUT/err.log
python3 -c "
import json; d=json.load(open('$OUT/bench.json')); pl=d['roofline']['per_layer']
print('bench', round(d['value']), round(d['ms_per_step'],4), d['parity']['bitexact'], [pl[i]['us_per_forward'] for i in (0,4,7,10)])"
