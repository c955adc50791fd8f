TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
summ() { python -c "
import json,sys
d=json.loads([l for l in open('$1') if l.startswith('{')][-1])
print('$1', round(d['value']), round(d['e2e']['value']), d['ms_per_step'], d.get('stages',{}).get('embedding'), d['clocks'])"; }
timeout 300 $TR --master-port 29517 tests/dist_sharded_check.py > gpurun_out/dist2.log 2>&1; echo rc=$?; grep bit-identical gpurun_out/dist2.log
timeout 400 $TR --master-port 29521 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/n2p.json 2> gpurun_out/n2p.err; summ gpurun_out/n2p.json
timeout 400 $TR --master-port 29522 bench.py --gpus 2 --steps 20 --warmup 5 --exchange nccl > gpurun_out/n2n.json 2> gpurun_out/n2n.err; summ gpurun_out/n2n.json
timeout 300 python bench.py --steps 20 --warmup 5 --cpu-seconds 1 > gpurun_out/n1.json 2>/dev/null; summ gpurun_out/n1.json
