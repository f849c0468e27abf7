#!/bin/bash
# compute-sanitizer over every kernel family + the randomised parity sweep.
set -u
OUT=gpurun_out/${1:-sanity}
mkdir -p $OUT
timeout 1500 compute-sanitizer --tool memcheck python tools/sanitize.py --big > $OUT/memcheck.log 2>&1; echo "rc=$?" >> $OUT/memcheck.log
timeout 1500 compute-sanitizer --tool racecheck python tools/sanitize.py > $OUT/racecheck.log 2>&1; echo "rc=$?" >> $OUT/racecheck.log
timeout 1500 python tools/parity_sweep.py 4242 300 > $OUT/parity_sweep.log 2>&1; echo "rc=$?" >> $OUT/parity_sweep.log
tail -4 $OUT/memcheck.log; grep -c "Race reported" $OUT/racecheck.log; tail -3 $OUT/racecheck.log; tail -3 $OUT/parity_sweep.log
