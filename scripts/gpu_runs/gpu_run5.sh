set -x
timeout 300 python -m pytest tests/test_gemm_gpu.py -x -q > gpurun_out/pytest_gemm.log 2>&1
timeout 600 python -m pytest tests/test_network_gpu.py -x -q > gpurun_out/pytest_net.log 2>&1
timeout 300 python -m pytest tests/test_dropin_gpu.py -x -q > gpurun_out/pytest_dropin.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --cpu-seconds 5 > gpurun_out/bench_mid.json 2> gpurun_out/bench_mid.err
echo done
