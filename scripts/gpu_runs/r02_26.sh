#!/bin/bash
# round 2, call 26: CTA-pair FM/LCB kernel -- first run against the debug library (mbarrier waits
# time out and trap instead of hanging), then parity with the release library, then timing A/B
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
LATTICE_LIB=$PWD/paper_2512_09200_b200/liblattice_b200_debug.so timeout 300 python -m pytest -q -x -p no:cacheprovider \
  "tests/test_fm_lcb_gpu.py::test_fm_lcb_exact_inputs_one_rounding[512-128-32-256-640-bf16]" > gpurun_out/r26_debug.log 2>&1
echo "debug rc=$?" >> gpurun_out/r26_debug.log
grep -q "debug rc=0" gpurun_out/r26_debug.log || exit 0
PARITY_LOG=gpurun_out/r26_parity.jsonl timeout 600 python -m pytest tests/test_fm_lcb_gpu.py -q -rA -p no:cacheprovider > gpurun_out/r26_fm.log 2>&1
echo "fm rc=$?" >> gpurun_out/r26_fm.log
timeout 300 python scripts/fm_bench.py large > gpurun_out/r26_bench_pair.log 2>&1
LATTICE_FM_PAIR=0 timeout 300 python scripts/fm_bench.py large > gpurun_out/r26_bench_single.log 2>&1
echo done
