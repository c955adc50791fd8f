nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2512_09200_b200/csrc -I include scripts/mma_probe.cu -o /tmp/mma_probe > /dev/null 2>&1
timeout 120 /tmp/mma_probe > gpurun_out/mma_probe.log 2>&1
timeout 300 python -m pytest tests/test_gemm_gpu.py -x -q > gpurun_out/pytest_gemm.log 2>&1
echo done
