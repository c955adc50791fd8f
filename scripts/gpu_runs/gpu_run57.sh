timeout 600 python -m pytest tests/test_network_gpu.py -x -q > gpurun_out/pytest_net.log 2>&1; echo rc=$?; tail -3 gpurun_out/pytest_net.log
