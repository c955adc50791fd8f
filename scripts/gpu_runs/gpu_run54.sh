summ() { python -c "
import json,sys
d=json.loads([l for l in open('$1') if l.startswith('{')][-1])
st=d.get('stages',{})
print('$1', round(d['value']), round(d['e2e']['value']), d['ms_per_step'], round(d['roofline']['frac'],3), st.get('embedding',{}).get('ms'), d['clocks'])"; }
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu2.log 2>&1; tail -2 gpurun_out/pytest_gpu2.log
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29591 bench.py --gpus 2 > gpurun_out/n2.json 2>/dev/null; summ gpurun_out/n2.json
timeout 300 python bench.py > gpurun_out/n1.json 2>/dev/null; summ gpurun_out/n1.json
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
