# full GPU suite after the JSONL work, drop-in driver, ingest bench, default bench line
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 300 tests/cpp/test_dropin > gpurun_out/dropin.log 2>&1; echo dropin rc=$?; tail -1 gpurun_out/dropin.log
timeout 600 python scripts/jsonl_bench.py 400000 40000 > gpurun_out/jsonl_bench.json 2>gpurun_out/jsonl_bench.err; echo jbench rc=$?; cat gpurun_out/jsonl_bench.json
timeout 400 python bench.py > gpurun_out/n1.json 2>gpurun_out/n1.err; echo bench rc=$?; tail -c 600 gpurun_out/n1.json
