#!/bin/bash
# round 2, call 51 (2 GPUs): the round-end sequence on the final code -- full GPU suite (multi-GPU
# tests active), smoke, the default 1-GPU bench line, and the driver's N=2 command
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
export PARITY_LOG=gpurun_out/parity_r02_51.jsonl
timeout 1500 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/pytest_r02_51.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r02_51.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02_51.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke_r02_51.log
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > gpurun_out/bench_r02_51.json 2> gpurun_out/bench_r02_51.err
echo "bench rc=$?" >> gpurun_out/bench_r02_51.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29751 \
    bench.py --gpus 2 > gpurun_out/bench_r02_51_n2.json 2> gpurun_out/bench_r02_51_n2.err
echo "bench n2 rc=$?" >> gpurun_out/bench_r02_51_n2.err
echo done
