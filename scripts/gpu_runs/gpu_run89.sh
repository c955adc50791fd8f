# peer owner pooling with the local source on the direct kernel: parity (Python + C++ sharded), A/B
timeout 900 python -m pytest tests/test_multi_gpu.py tests/test_dropin_gpu.py -x -q > gpurun_out/pytest_local.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_local.log
summ() { python -c "
import json,sys
d=json.loads([l for l in open('$1') if l.startswith('{')][-1])
e=d['stages']['embedding']
print('$1', round(d['value']), d['ms_per_step'], 'owner', [round(x,3) for x in e.get('peer_split_ms',[])], d['clocks']['sm_mhz'])"; }
for v in 0 1 0 1; do
  LATTICE_PEER_LOCAL=$v timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29661 bench.py --gpus 2 --cpu-seconds 0.1 > gpurun_out/n2_local$v.json 2>/dev/null; summ gpurun_out/n2_local$v.json
done | tee gpurun_out/peer_local_ab.log
