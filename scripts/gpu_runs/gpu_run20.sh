set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python scripts/bag_sweep.py l2 > gpurun_out/bag_l2.log 2>&1
cat gpurun_out/bag_l2.log
echo done
