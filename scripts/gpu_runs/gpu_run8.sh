set -x
timeout 600 python -m pytest tests/test_multi_gpu.py -x -q > gpurun_out/pytest_multi.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/bench_mid_n2.json 2> gpurun_out/bench_mid_n2.err
echo done
