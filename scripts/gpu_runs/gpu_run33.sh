summ() { python -c "
import json,sys
d=json.loads([l for l in open('$1') if l.startswith('{')][-1])
print('$1', round(d['value']), round(d['e2e']['value']), round(d['roofline']['frac'],3), d.get('stages',{}).get('embedding',{}).get('ms'), d.get('stages',{}).get('embedding',{}).get('peer_split_ms'), d['clocks'])"; }
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu2.log 2>&1; tail -2 gpurun_out/pytest_gpu2.log
timeout 300 python bench.py > gpurun_out/n1.json 2>/dev/null; summ gpurun_out/n1.json
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 2 > gpurun_out/n2.json 2>/dev/null; summ gpurun_out/n2.json
timeout 300 python bench.py --workload micro --dtype bf16 --cpu-seconds 2 > gpurun_out/mb.json 2>/dev/null; summ gpurun_out/mb.json
timeout 300 python bench.py --workload micro --dtype f32 --cpu-seconds 2 > gpurun_out/mf.json 2>/dev/null; summ gpurun_out/mf.json
