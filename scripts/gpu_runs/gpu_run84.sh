# PDL on the 2-GPU peer path: sharded parity (bit-identical to 1 GPU), C++ ShardedNetwork, N=2 bench
timeout 900 python -m pytest tests/test_multi_gpu.py tests/test_dropin_gpu.py -x -q > gpurun_out/pytest_mgpu.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_mgpu.log
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 > gpurun_out/n2.json 2>gpurun_out/n2.err; python -c "
import json
d=json.loads([l for l in open('gpurun_out/n2.json') if l.startswith('{')][-1])
print(round(d['value']), round(d['e2e']['value']), d['ms_per_step'], d['clocks']['sm_mhz'])"
