# bag kernel variants after the instruction diet (env knobs only), same box
summ() { python -c "
import json,sys
d=json.loads([l for l in open('$1') if l.startswith('{')][-1])
print('$2', round(d['value']), d['ms_per_step'], 'emb', round(d['stages']['embedding']['ms'],3), d['clocks']['sm_mhz'])"; }
for v in 0 2 1 0 2; do
  LATTICE_BAG_VARIANT=$v timeout 200 python bench.py --steps 40 --warmup 5 --cpu-seconds 0.1 > gpurun_out/bagv$v.json 2>/dev/null; summ gpurun_out/bagv$v.json variant$v
done | tee gpurun_out/bag_variant_ab.log
