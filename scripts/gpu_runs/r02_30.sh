#!/bin/bash
# round 2, call 30: K2 suite with the single-CTA large kernel's warp-collective fix (default) and the
# opt-in pair kernel (subprocess), network suite, K2 timing
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
PARITY_LOG=gpurun_out/r30_parity.jsonl timeout 900 python -m pytest tests/test_fm_lcb_gpu.py tests/test_network_gpu.py -q -rA -p no:cacheprovider > gpurun_out/r30_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r30_tests.log
timeout 300 python scripts/fm_bench.py > gpurun_out/r30_fm_bench_single.log 2>&1
LATTICE_FM_PAIR=1 timeout 300 python scripts/fm_bench.py large > gpurun_out/r30_fm_bench_pair.log 2>&1
echo done
