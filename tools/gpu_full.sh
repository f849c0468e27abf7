#!/bin/bash
# Full evidence run: GPU tests, smoke, bench line (CPU baseline + e2e + parity),
# reference arm, ncu launch list, ncu --set full of K0/K1/GEMM on the first
# 56x56 layer and the first 7x7 layer.  Usage: gpu_full.sh TAG
set -u
TAG=${1:-full}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q --durations 15 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-verify > $OUT/ncu_launch.log 2>&1
for L in 0 10; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"input_range|input_quant|gemm_epilogue" -s 9 -c 3 \
    -o $OUT/prof_L$L python bench.py --layers $L --steps 1 --warmup 3 --no-cpu --no-e2e --no-verify > $OUT/ncu_L$L.log 2>&1
done
tail -3 $OUT/pytest_gpu.log; tail -2 $OUT/smoke.log
python3 -c "
import json; d=json.load(open('$OUT/bench.json')); print(round(d['value']), d['ms_per_step'], d['parity']['bitexact'], d['e2e']['value'], d['roofline']['frac'])
for l in d['roofline']['per_layer']: print(l)"
head -c 600 $OUT/bench_ref.json
du -sh $OUT/* | sort -h | tail -8
# keep the merge-back under gpurun's 64 MiB cap: summaries first, big reps last to go
for f in $OUT/prof_L0.ncu-rep $OUT/prof_L10.ncu-rep; do
  [ -f $f ] && ncu -i $f --page raw --csv > ${f%.ncu-rep}_raw.csv 2>/dev/null
done
tot=$(du -sm $OUT | cut -f1); if [ $tot -gt 60 ]; then rm -f $OUT/prof_L0.ncu-rep; fi
tot=$(du -sm $OUT | cut -f1); if [ $tot -gt 60 ]; then rm -f $OUT/prof_L10.ncu-rep; fi
du -sh $OUT
