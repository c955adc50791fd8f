#!/bin/bash
# round 2, call 4: full GPU suite (fp64 drop-in numerics, concurrency/cooperative GEMM, wide hidden
# rows, drop-in C++ edge cases), smoke, and a short mid bench (graph capture of cooperative launches)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
export PARITY_LOG=gpurun_out/parity_r02_04.jsonl
rm -f $PARITY_LOG
timeout 1500 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/pytest_r02_04.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r02_04.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02_04.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke_r02_04.log
timeout 600 python bench.py --steps 20 --warmup 5 --cpu-seconds 5 > gpurun_out/bench_r02_04.json 2> gpurun_out/bench_r02_04.err
echo "bench rc=$?" >> gpurun_out/bench_r02_04.err
