OUT=gpurun_out/band2; mkdir -p $OUT
for cfg in "" "LANCE_BAND_K0=1" "LANCE_BAND_K1=1" "LANCE_BAND_K0=1 LANCE_BAND_K1=1"; do
  echo "== $cfg" >> $OUT/exp.txt
  env $cfg timeout 120 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > $OUT/b.json 2>> $OUT/exp.err
  python -c "
import json; d=json.load(open('$OUT/b.json')); print('  value', round(d['value']))
seen=set()
for l in d['roofline']['per_layer']:
    if l['c'] in seen: continue
    seen.add(l['c']); print('  ', l['c'], l['h'], l['us_per_forward'])" >> $OUT/exp.txt
done
