# final 4-GPU check of the committed state: sharded parity + mid N=4 bench
timeout 600 python -m pytest tests/test_multi_gpu.py -x -q > gpurun_out/pytest_mgpu4.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_mgpu4.log
timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29671 bench.py --gpus 4 > gpurun_out/final_n4.json 2>gpurun_out/final_n4.err; echo bench rc=$?
python -c "
import json
d=json.loads([l for l in open('gpurun_out/final_n4.json') if l.startswith('{')][-1])
print(round(d['value']), round(d['e2e']['value']), d['ms_per_step'], d['clocks']['sm_mhz'])"
timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29672 bench.py --gpus 4 --impl reference > gpurun_out/final_n4_ref.json 2>/dev/null; echo ref rc=$?; tail -c 150 gpurun_out/final_n4_ref.json
