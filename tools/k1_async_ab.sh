OUT=gpurun_out/k1a; mkdir -p $OUT
LANCE_K1_ASYNC=4 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "golden or random" > $OUT/t_async4.log 2>&1; echo rc=$? >> $OUT/t_async4.log
for rep in 1 2; do
for cfg in "" "LANCE_K1_ASYNC=4"; do
  echo "== $cfg" >> $OUT/exp.txt
  env $cfg timeout 120 python bench.py --layers 0,4,7,10 --steps 5 --warmup 3 --no-cpu --no-e2e > $OUT/b.json 2>> $OUT/exp.err
  python -c "
import json; d=json.load(open('$OUT/b.json'))
for l in d['roofline']['per_layer']: print('  ', l['c'], l['h'], l['us_per_forward'])" >> $OUT/exp.txt
done
done
