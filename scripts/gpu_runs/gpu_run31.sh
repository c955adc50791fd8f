B="python bench.py --steps 10 --warmup 3 --cpu-seconds 1"
summ() { python -c "
import json,sys
d=json.loads([l for l in open('$1') if l.startswith('{')][-1])
print('$1', round(d['value']), round(d['roofline']['frac'],3), d.get('stages',{}).get('embedding',{}).get('ms'), d.get('stages',{}).get('embedding',{}).get('peer_split_ms'), d['clocks']['sm_mhz'])"; }
for k in 1 0; do for v in 2 0; do
export LATTICE_BAG_V3=$k LATTICE_BAG_VARIANT=$v
timeout 300 python bench.py --workload micro --dtype bf16 --steps 20 --warmup 3 --cpu-seconds 1 > gpurun_out/mb_k${k}v$v.json 2>/dev/null; summ gpurun_out/mb_k${k}v$v.json
timeout 300 python bench.py --workload micro --dtype f32 --steps 20 --warmup 3 --cpu-seconds 1 > gpurun_out/mf_k${k}v$v.json 2>/dev/null; summ gpurun_out/mf_k${k}v$v.json
timeout 300 $B > gpurun_out/n1_k${k}v$v.json 2>/dev/null; summ gpurun_out/n1_k${k}v$v.json
timeout 300 $B --exchange peer1 > gpurun_out/n1p_k${k}v$v.json 2>/dev/null; summ gpurun_out/n1p_k${k}v$v.json
done; done
