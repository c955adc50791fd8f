summ() { python -c "
import json,sys
d=json.loads([l for l in open('$1') if l.startswith('{')][-1])
print('$1', round(d['value']), round(d['e2e']['value']), d['ms_per_step'], d.get('stages',{}).get('embedding'), d['clocks'])"; }
for n in 4 2; do
timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2953$n bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/n${n}p.json 2> gpurun_out/n${n}p.err; summ gpurun_out/n${n}p.json
done
timeout 300 python bench.py --steps 20 --warmup 5 --cpu-seconds 1 > gpurun_out/n1.json 2>/dev/null; summ gpurun_out/n1.json
