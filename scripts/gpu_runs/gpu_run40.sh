summ() { python -c "
import json,sys
d=json.loads([l for l in open('$1') if l.startswith('{')][-1])
st=d.get('stages',{})
print('$1', round(d['value']), round(d['e2e']['value']), d['ms_per_step'], st.get('embedding',{}).get('ms'), d['gpu_launches'], d['clocks']['sm_mhz'])"; }
timeout 300 python bench.py --workload full --steps 20 --warmup 5 --cpu-seconds 1 > gpurun_out/full_n1.json 2>gpurun_out/full_n1.err; summ gpurun_out/full_n1.json; tail -3 gpurun_out/full_n1.err
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 2 > gpurun_out/n2.json 2>gpurun_out/n2.err; summ gpurun_out/n2.json; tail -3 gpurun_out/n2.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29562 bench.py --gpus 2 --workload full --steps 10 --warmup 3 > gpurun_out/full_n2.json 2>gpurun_out/full_n2.err; summ gpurun_out/full_n2.json; tail -3 gpurun_out/full_n2.err
timeout 300 python -m pytest tests/test_multi_gpu.py -x -q 2>&1 | tail -2
