OUT=gpurun_out/rsab; mkdir -p $OUT
for rep in 1 2; do
for cfg in "" "LANCE_RS_GEMM=1"; do
  echo "== $cfg" >> $OUT/exp.txt
  env $cfg timeout 120 python bench.py --layers 0,4,7,10 --steps 5 --warmup 3 --no-cpu --no-e2e > $OUT/b.json 2>> $OUT/exp.err
  python -c "
import json; d=json.load(open('$OUT/b.json'))
for l in d['roofline']['per_layer']: print('  ', l['c'], l['h'], l['us_per_forward'], round(sum(l['us_per_forward']),1))" >> $OUT/exp.txt
done
done
