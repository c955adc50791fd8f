#!/bin/bash
# round 2, call 20 (2 GPUs): e2e replaying the forward from a graph per input buffer: default bench
# on one GPU, mid and full at N=2
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --no-micro > gpurun_out/bench20_n1.json 2> gpurun_out/bench20_n1.err
echo "rc=$?" >> gpurun_out/bench20_n1.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29911 \
    bench.py --gpus 2 > gpurun_out/bench20_mid_n2.json 2> gpurun_out/bench20_mid_n2.err
echo "rc=$?" >> gpurun_out/bench20_mid_n2.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29912 \
    bench.py --gpus 2 --workload full > gpurun_out/bench20_full_n2.json 2> gpurun_out/bench20_full_n2.err
echo "rc=$?" >> gpurun_out/bench20_full_n2.err
