summ() { python -c "
import json,sys
d=json.loads([l for l in open('$1') if l.startswith('{')][-1])
st=d.get('stages',{})
print('$1', round(d['value']), d['ms_per_step'], st.get('embedding',{}).get('ms'), st.get('fm_lcb',{}).get('ms_per_block'), st.get('mlp',{}).get('ms_per_block'), d['clocks']['sm_mhz'])"; }
timeout 600 python -m pytest tests/test_network_gpu.py -x -q > gpurun_out/pytest_net.log 2>&1; echo rc=$?; tail -15 gpurun_out/pytest_net.log
timeout 900 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2 --master-port 29603 bench.py --gpus 2 --workload large --steps 10 --warmup 3 > gpurun_out/large_n2.json 2>gpurun_out/large_n2.err; summ gpurun_out/large_n2.json
