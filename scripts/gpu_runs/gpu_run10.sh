set -x
timeout 300 python -m pytest tests/test_embedding_bag_gpu.py tests/test_network_gpu.py -x -q > gpurun_out/pytest_bag.log 2>&1
timeout 900 python scripts/bag_sweep.py > gpurun_out/bag_sweep.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --cpu-seconds 3 > gpurun_out/bench_mid.json 2> gpurun_out/bench_mid.err
echo done
