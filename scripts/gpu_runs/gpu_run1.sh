set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_micro_f32.json 2> gpurun_out/bench_micro_f32.err
python bench.py --steps 20 --warmup 5 --dtype bf16 --cpu-seconds 5 > gpurun_out/bench_micro_bf16.json 2> gpurun_out/bench_micro_bf16.err
python bench.py --steps 3 --warmup 3 --cpu-seconds 1 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --cpu-seconds 1 > gpurun_out/ncu.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:bag_kernel -s 3 -c 1 -o gpurun_out/prof_bag python bench.py --steps 3 --warmup 3 --cpu-seconds 1 > gpurun_out/ncu_full.log 2>&1
echo done
