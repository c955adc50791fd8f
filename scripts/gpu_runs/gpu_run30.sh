B="python bench.py --steps 10 --warmup 3 --cpu-seconds 1"
summ() { python -c "
import json,sys
d=json.loads([l for l in open('$1') if l.startswith('{')][-1])
print('$1', round(d['value']), d['roofline']['frac'], d.get('stages',{}).get('embedding',{}).get('ms'), d.get('stages',{}).get('embedding',{}).get('peer_split_ms'), d['clocks']['sm_mhz'])"; }
timeout 600 python -m pytest tests/test_embedding_bag_gpu.py tests/test_network_gpu.py -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for v in 2 1 0; do
LATTICE_BAG_VARIANT=$v timeout 300 $B > gpurun_out/n1_v$v.json 2>/dev/null; summ gpurun_out/n1_v$v.json
LATTICE_BAG_VARIANT=$v timeout 300 $B --exchange peer1 > gpurun_out/n1p_v$v.json 2>/dev/null; summ gpurun_out/n1p_v$v.json
LATTICE_BAG_VARIANT=$v timeout 300 python bench.py --workload micro --dtype bf16 --steps 20 --warmup 3 --cpu-seconds 1 > gpurun_out/mb_v$v.json 2>/dev/null; summ gpurun_out/mb_v$v.json
LATTICE_BAG_VARIANT=$v timeout 300 python bench.py --workload micro --dtype f32 --steps 20 --warmup 3 --cpu-seconds 1 > gpurun_out/mf_v$v.json 2>/dev/null; summ gpurun_out/mf_v$v.json
done
