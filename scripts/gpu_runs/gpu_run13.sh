set -x
timeout 300 python -m pytest tests/test_gemm_gpu.py tests/test_network_gpu.py -x -q > gpurun_out/pytest_gemm.log 2>&1 || exit 1
timeout 600 python bench.py --steps 20 --warmup 5 --cpu-seconds 3 > gpurun_out/bench_mid.json 2> gpurun_out/bench_mid.err
timeout 300 python bench.py --steps 3 --warmup 3 --cpu-seconds 1 > gpurun_out/plain_mid.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_mid.csv python bench.py --steps 3 --warmup 3 --cpu-seconds 1 > gpurun_out/ncu_mid.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 1 -c 1 -o gpurun_out/prof_gemm_g2 python bench.py --steps 3 --warmup 3 --cpu-seconds 1 > gpurun_out/ncu_gemm.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fm_lcb -s 4 -c 1 -o gpurun_out/prof_fm3 python bench.py --steps 3 --warmup 3 --cpu-seconds 1 > gpurun_out/ncu_fm.log 2>&1
echo done
