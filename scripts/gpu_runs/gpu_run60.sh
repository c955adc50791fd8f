summ() { python -c "
import json,sys
d=json.loads([l for l in open('$1') if l.startswith('{')][-1])
print('$1', round(d['value']), round(d['e2e']['value']), d['ms_per_step'], d['config'].get('launch'), d['clocks']['sm_mhz'])"; }
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 > gpurun_out/n2.json 2>gpurun_out/n2.err; summ gpurun_out/n2.json; tail -3 gpurun_out/n2.err
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 --no-graph > gpurun_out/n2e.json 2>/dev/null; summ gpurun_out/n2e.json
timeout 300 python bench.py --workload full --steps 20 --warmup 5 --cpu-seconds 1 > gpurun_out/full.json 2>gpurun_out/full.err; summ gpurun_out/full.json; tail -3 gpurun_out/full.err
timeout 300 python bench.py > gpurun_out/n1.json 2>/dev/null; summ gpurun_out/n1.json
