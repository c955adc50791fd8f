#!/bin/bash
# round 2, call 29: pair kernel with relaxed drained-arrivals and a register-prefetched partner residual
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_fm_lcb_gpu.py -q -rA -p no:cacheprovider -k "512 or 384 or 400" > gpurun_out/r29_fm.log 2>&1
echo "fm rc=$?" >> gpurun_out/r29_fm.log
grep -q "fm rc=0" gpurun_out/r29_fm.log || exit 0
timeout 300 python scripts/fm_bench.py large > gpurun_out/r29_bench_pair.log 2>&1
LATTICE_FM_TRACE=1 timeout 120 python scripts/fm_bench.py large 2>&1 | tail -14 > gpurun_out/r29_trace.log
echo done
