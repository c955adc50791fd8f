timeout 300 ./tests/cpp/test_sharded 2 > gpurun_out/cpp_sharded.log 2>&1; echo rc=$?; cat gpurun_out/cpp_sharded.log | tail -5
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu2.log 2>&1; tail -3 gpurun_out/pytest_gpu2.log
