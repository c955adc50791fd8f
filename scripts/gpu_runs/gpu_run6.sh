set -x
timeout 300 python -m pytest tests/test_embedding_bag_gpu.py tests/test_network_gpu.py -x -q > gpurun_out/pytest_bag.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --cpu-seconds 3 > gpurun_out/bench_mid.json 2> gpurun_out/bench_mid.err
timeout 600 python bench.py --workload micro --steps 50 --warmup 5 --cpu-seconds 2 > gpurun_out/bench_micro_f32.json 2> gpurun_out/bench_micro_f32.err
timeout 600 python bench.py --workload micro --dtype bf16 --steps 50 --warmup 5 --cpu-seconds 2 > gpurun_out/bench_micro_bf16.json 2> gpurun_out/bench_micro_bf16.err
echo done
