set -x
timeout 300 python -m pytest tests/test_zipper_gpu.py -x -q > gpurun_out/pytest_zip.log 2>&1
timeout 600 python bench.py --workload full --steps 20 --warmup 5 --cpu-seconds 3 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 300 python bench.py --steps 3 --warmup 3 --cpu-seconds 1 > gpurun_out/plain_mid.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_mid.csv python bench.py --steps 3 --warmup 3 --cpu-seconds 1 > gpurun_out/ncu_mid.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 0 -c 3 -o gpurun_out/prof_gemm_mlp python bench.py --steps 3 --warmup 3 --cpu-seconds 1 > gpurun_out/ncu_gemm.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fm_lcb -s 4 -c 1 -o gpurun_out/prof_fm4 python bench.py --steps 3 --warmup 3 --cpu-seconds 1 > gpurun_out/ncu_fm.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:bag_kernel -s 2 -c 1 -o gpurun_out/prof_bag3 python bench.py --steps 3 --warmup 3 --cpu-seconds 1 > gpurun_out/ncu_bag.log 2>&1
echo done
