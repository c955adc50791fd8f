timeout 600 python -m pytest tests/test_jsonl_gpu.py -x -q > gpurun_out/pytest_jsonl.log 2>&1; echo jsonl rc=$?; tail -2 gpurun_out/pytest_jsonl.log
timeout 600 python scripts/jsonl_bench.py 400000 40000 > gpurun_out/jsonl_bench.json 2>gpurun_out/jsonl_bench.err; echo bench rc=$?; cat gpurun_out/jsonl_bench.json; tail -3 gpurun_out/jsonl_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/jsonl_launches.csv python scripts/jsonl_bench.py 400000 100 > /dev/null 2>&1; echo ncu rc=$?
