# final multi-GPU record (PDL, bucket, st256 all in): mid N=2/4 + parity; micro bf16 on 1 GPU
timeout 900 python -m pytest tests/test_multi_gpu.py -x -q > gpurun_out/pytest_mgpu4.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_mgpu4.log
summ() { python -c "
import json,sys
d=json.loads([l for l in open('$1') if l.startswith('{')][-1])
print('$1', round(d['value']), round(d['e2e']['value']), d['ms_per_step'], d['clocks']['sm_mhz'])"; }
CUDA_VISIBLE_DEVICES=0 timeout 400 python bench.py > gpurun_out/final_n1.json 2>/dev/null; summ gpurun_out/final_n1.json
for n in 2 4; do
timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2963$n bench.py --gpus $n > gpurun_out/final_n$n.json 2>gpurun_out/final_n$n.err; summ gpurun_out/final_n$n.json
done
CUDA_VISIBLE_DEVICES=0 timeout 400 python bench.py --workload micro --dtype bf16 > gpurun_out/final_micro_bf16.json 2>/dev/null; summ gpurun_out/final_micro_bf16.json
