summ() { python -c "
import json,sys
d=json.loads([l for l in open('$1') if l.startswith('{')][-1])
st=d.get('stages',{})
print('$1', round(d['value']), d['ms_per_step'], st.get('embedding',{}).get('ms'), st.get('mlp',{}).get('ms_per_block'), st.get('fm_lcb',{}).get('ms_per_block'), st.get('tower',{}).get('ms'), d['clocks']['sm_mhz'])"; }
for k in 0 3 1 0 3; do
LATTICE_BAG_L2KEEP=$k timeout 300 python bench.py --steps 20 --warmup 5 --cpu-seconds 1 > gpurun_out/n1_k$k.json 2>/dev/null; summ gpurun_out/n1_k$k.json
done
for k in 0 3; do
LATTICE_BAG_L2KEEP=$k timeout 300 python bench.py --workload micro --dtype bf16 --steps 20 --warmup 5 --cpu-seconds 1 > gpurun_out/mb_k$k.json 2>/dev/null; summ gpurun_out/mb_k$k.json
LATTICE_BAG_L2KEEP=$k timeout 300 python bench.py --workload micro --dtype f32 --steps 20 --warmup 5 --cpu-seconds 1 > gpurun_out/mf_k$k.json 2>/dev/null; summ gpurun_out/mf_k$k.json
done
