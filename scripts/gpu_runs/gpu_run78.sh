# 4 GPUs: sharded parity, mid / large / full benches (peer exchange), scaling record
timeout 900 python -m pytest tests/test_multi_gpu.py -x -q > gpurun_out/pytest_mgpu4.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_mgpu4.log
summ() { python -c "
import json,sys
d=json.loads([l for l in open('$1') if l.startswith('{')][-1])
st=d.get('stages',{})
print('$1', round(d['value']), round(d['e2e']['value']), d['ms_per_step'], 'emb', st.get('embedding',{}).get('ms'), 'fm', st.get('fm_lcb',{}).get('ms_per_block'), d['clocks']['sm_mhz'])"; }
for n in 2 4; do
timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2961$n bench.py --gpus $n > gpurun_out/mid_n$n.json 2>gpurun_out/mid_n$n.err; summ gpurun_out/mid_n$n.json
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29621 bench.py --gpus 4 --workload large --steps 10 --warmup 3 > gpurun_out/large_n4.json 2>gpurun_out/large_n4.err; summ gpurun_out/large_n4.json; tail -2 gpurun_out/large_n4.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29622 bench.py --gpus 4 --workload full --steps 10 --warmup 3 > gpurun_out/full_n4.json 2>gpurun_out/full_n4.err; summ gpurun_out/full_n4.json; tail -2 gpurun_out/full_n4.err
