for i in 1 2; do timeout 600 python scripts/jsonl_bench.py 400000 40000 2>/dev/null; done | tee gpurun_out/jsonl_bench.json
