summ() { python -c "
import json,sys
d=json.loads([l for l in open('$1') if l.startswith('{')][-1])
print('$1', round(d['value']), round(d['e2e']['value']), d['ms_per_step'], round(d['roofline']['frac'],3), d['stages']['embedding'], d['clocks'])"; }
for n in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2957$n bench.py --gpus $n --workload large --steps 10 --warmup 3 > gpurun_out/large_n$n.json 2> gpurun_out/large_n$n.err; echo rc=$?; summ gpurun_out/large_n$n.json; tail -3 gpurun_out/large_n$n.err
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29579 bench.py --gpus 4 --workload full --steps 10 --warmup 3 > gpurun_out/full_n4.json 2> gpurun_out/full_n4.err; echo rc=$?; summ gpurun_out/full_n4.json; tail -3 gpurun_out/full_n4.err
nvidia-smi --query-gpu=memory.used,memory.total --format=csv
