timeout 300 tests/cpp/test_dropin > gpurun_out/dropin.log 2>&1; echo dropin rc=$?; tail -3 gpurun_out/dropin.log
timeout 600 python scripts/jsonl_bench.py 400000 40000 > gpurun_out/jsonl_bench.json 2>gpurun_out/jsonl_bench.err; echo bench rc=$?; cat gpurun_out/jsonl_bench.json; tail -3 gpurun_out/jsonl_bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pass1_kernel -c 1 -o gpurun_out/prof_jsonl_pass1 python scripts/jsonl_bench.py 100000 100 > gpurun_out/ncu_jsonl.log 2>&1; echo ncu rc=$?
