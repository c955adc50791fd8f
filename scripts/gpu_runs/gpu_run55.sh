summ() { python -c "
import json,sys
d=json.loads([l for l in open('$1') if l.startswith('{')][-1])
st=d.get('stages',{})
print('$1', round(d['value']), round(d['e2e']['value']), d['ms_per_step'], round(d['roofline']['frac'],3), st.get('embedding',{}).get('ms'), st.get('fm_lcb',{}).get('ms_per_block'), st.get('mlp',{}).get('ms_per_block'), d['clocks']['sm_mhz'])"; }
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 python bench.py --workload full --steps 20 --warmup 5 --cpu-seconds 1 > gpurun_out/full_n1.json 2>/dev/null; summ gpurun_out/full_n1.json
timeout 900 $T --nproc-per-node 4 --master-port 29601 bench.py --gpus 4 --workload large --steps 10 --warmup 3 > gpurun_out/large_n4.json 2>/dev/null; summ gpurun_out/large_n4.json
timeout 900 $T --nproc-per-node 4 --master-port 29602 bench.py --gpus 4 --workload full --steps 10 --warmup 3 > gpurun_out/full_n4.json 2>/dev/null; summ gpurun_out/full_n4.json
timeout 900 $T --nproc-per-node 2 --master-port 29603 bench.py --gpus 2 --workload large --steps 10 --warmup 3 > gpurun_out/large_n2.json 2>/dev/null; summ gpurun_out/large_n2.json
timeout 600 $T --nproc-per-node 4 --master-port 29604 bench.py --gpus 4 > gpurun_out/n4.json 2>/dev/null; summ gpurun_out/n4.json
