set -x
timeout 300 python -m pytest tests/test_gemm_gpu.py tests/test_network_gpu.py -x -q > gpurun_out/pytest_gemm.log 2>&1
timeout 900 python scripts/bag_sweep.py > gpurun_out/bag_sweep.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --cpu-seconds 3 > gpurun_out/bench_mid.json 2> gpurun_out/bench_mid.err
timeout 300 python bench.py --steps 3 --warmup 3 --cpu-seconds 1 > gpurun_out/plain_mid.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_mid.csv python bench.py --steps 3 --warmup 3 --cpu-seconds 1 > gpurun_out/ncu_mid.log 2>&1
echo done
