set -x
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_mid.json 2> gpurun_out/bench_mid.err
python bench.py --steps 3 --warmup 3 --cpu-seconds 1 > gpurun_out/plain_mid.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_mid.csv python bench.py --steps 3 --warmup 3 --cpu-seconds 1 > gpurun_out/ncu_mid.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 20 -c 3 -o gpurun_out/prof_gemm python bench.py --steps 3 --warmup 3 --cpu-seconds 1 > gpurun_out/ncu_gemm.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fm_lcb -s 2 -c 1 -o gpurun_out/prof_fm python bench.py --steps 3 --warmup 3 --cpu-seconds 1 > gpurun_out/ncu_fm.log 2>&1
echo done
