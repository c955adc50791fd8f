set -x
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --cpu-seconds 3 > gpurun_out/bench_mid.json 2> gpurun_out/bench_mid.err
echo done
