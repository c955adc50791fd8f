set -x
timeout 300 python -m pytest tests/test_gemm_gpu.py -x -q > gpurun_out/pytest_gemm.log 2>&1
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
python bench.py --steps 50 --warmup 5 > gpurun_out/bench_micro_f32.json 2> gpurun_out/bench_micro_f32.err
python bench.py --steps 50 --warmup 5 --dtype bf16 --cpu-seconds 5 > gpurun_out/bench_micro_bf16.json 2> gpurun_out/bench_micro_bf16.err
echo done
