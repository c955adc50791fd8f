# JSONL ingest: GPU parity vs the reference (golden + live), then the full GPU suite
timeout 900 python -m pytest tests/test_jsonl_gpu.py -x -q > gpurun_out/pytest_jsonl.log 2>&1; echo jsonl rc=$?; tail -25 gpurun_out/pytest_jsonl.log
