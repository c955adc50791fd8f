set -x
nvidia-smi topo -m | head -5
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 tests/dist_sharded_check.py > gpurun_out/dist2.log 2>&1; echo rc=$?; tail -5 gpurun_out/dist2.log
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/bench_n2_peer.json 2> gpurun_out/bench_n2_peer.err; echo rc=$?; tail -c 1500 gpurun_out/bench_n2_peer.json; tail -5 gpurun_out/bench_n2_peer.err
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29519 bench.py --gpus 2 --steps 20 --warmup 5 --exchange nccl > gpurun_out/bench_n2_nccl.json 2> gpurun_out/bench_n2_nccl.err; echo rc=$?
echo done
