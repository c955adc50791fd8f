# bag L2 policy re-check on the final code (bit 0: rows evict_last, bit 1: outputs evict_first)
summ() { python -c "
import json,sys
d=json.loads([l for l in open('$1') if l.startswith('{')][-1])
print('$2', round(d['value']), d['ms_per_step'], 'emb', round(d['stages']['embedding']['ms'],3), 'dense', round(d['stages']['dense_total']['ms'],3), d['clocks']['sm_mhz'])"; }
for v in 3 1 0 2 3 1; do
  LATTICE_BAG_L2KEEP=$v timeout 200 python bench.py --steps 40 --warmup 5 --cpu-seconds 0.1 > gpurun_out/l2k$v.json 2>/dev/null; summ gpurun_out/l2k$v.json l2keep$v
done | tee gpurun_out/l2keep_ab.log
