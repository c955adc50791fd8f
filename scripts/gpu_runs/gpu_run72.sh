# 2 GPUs: sharded parity (peer + NCCL paths), C++ ShardedNetwork test, mid bench N=2
timeout 900 python -m pytest tests/test_multi_gpu.py tests/test_dropin_gpu.py -x -q > gpurun_out/pytest_mgpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_mgpu.log
summ() { python -c "
import json,sys
d=json.loads([l for l in open('$1') if l.startswith('{')][-1])
print('$1', round(d['value']), round(d['e2e']['value']), d['ms_per_step'], d['clocks']['sm_mhz'])"; }
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 > gpurun_out/n2.json 2>gpurun_out/n2.err; summ gpurun_out/n2.json; tail -2 gpurun_out/n2.err
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 --impl reference > gpurun_out/n2ref.json 2>/dev/null; tail -c 300 gpurun_out/n2ref.json
