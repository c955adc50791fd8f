timeout 900 python -m pytest tests/test_ktap_gpu.py tests/test_dense_gpu.py tests/test_objective_gpu.py -x -q > gpurun_out/pytest_k.log 2>&1; tail -15 gpurun_out/pytest_k.log
