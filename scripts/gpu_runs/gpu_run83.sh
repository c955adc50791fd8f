# PDL A/B, alternating order
summ() { python -c "
import json,sys
d=json.loads([l for l in open('$1') if l.startswith('{')][-1])
print('$1', round(d['value']), round(d['e2e']['value']), d['ms_per_step'], d['clocks']['sm_mhz'])"; }
for v in 1 0 0 1 1 0; do
  LATTICE_PDL=$v timeout 300 python bench.py --steps 40 --warmup 5 --cpu-seconds 0.1 > gpurun_out/mid_pdl$v.json 2>/dev/null; summ gpurun_out/mid_pdl$v.json
done | tee gpurun_out/pdl_ab2.log
