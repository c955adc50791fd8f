# staged (peer) bag kernel: magic-number chunk decode; parity at N=2, then A/B of the owner kernel
timeout 900 python -m pytest tests/test_multi_gpu.py tests/test_embedding_bag_gpu.py -x -q > gpurun_out/pytest_staged.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_staged.log
summ() { python -c "
import json,sys
d=json.loads([l for l in open('$1') if l.startswith('{')][-1])
e=d['stages']['embedding']
print('$1', round(d['value']), d['ms_per_step'], 'owner', [round(x,3) for x in e.get('peer_split_ms',[])], d['clocks']['sm_mhz'])"; }
for v in base new base new; do
  if [ $v = base ]; then export LATTICE_LIB=$PWD/ab/base.so; else unset LATTICE_LIB; fi
  timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29651 bench.py --gpus 2 --cpu-seconds 0.1 > gpurun_out/n2_$v.json 2>/dev/null; summ gpurun_out/n2_$v.json
done | tee gpurun_out/staged_ab.log
