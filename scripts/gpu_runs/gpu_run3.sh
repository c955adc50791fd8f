set -x
timeout 600 python -m pytest tests/test_network_gpu.py -x -q > gpurun_out/pytest_net.log 2>&1
timeout 300 python -m pytest tests/test_gemm_gpu.py tests/test_zipper_gpu.py -q > gpurun_out/pytest_gemm_zip.log 2>&1
echo done
