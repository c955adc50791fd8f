timeout 900 python -m pytest tests/test_network_gpu.py tests/test_dropin_gpu.py -x -q > gpurun_out/pytest_check.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_check.log
timeout 300 tests/cpp/test_dropin > gpurun_out/dropin.log 2>&1; echo dropin rc=$?; tail -2 gpurun_out/dropin.log
