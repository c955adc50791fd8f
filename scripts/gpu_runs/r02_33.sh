#!/bin/bash
# round 2, call 33 (2 GPUs): the driver's exact commands at N=2 -- reference arm first, then ours
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 \
    bench.py --impl reference --gpus 2 --steps 10 --warmup 3 > gpurun_out/r33_ref_n2.json 2> gpurun_out/r33_ref_n2.err
echo "ref rc=$?" >> gpurun_out/r33_ref_n2.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 \
    bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/r33_n2.json 2> gpurun_out/r33_n2.err
echo "ours rc=$?" >> gpurun_out/r33_n2.err
echo done
