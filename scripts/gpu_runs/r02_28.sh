#!/bin/bash
# round 2, call 28: K2 suite (pair kernel + fixed single-CTA large kernel), pair vs single timing,
# wait-site trace, and one ncu capture of the pair kernel
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
PARITY_LOG=gpurun_out/r28_parity.jsonl timeout 600 python -m pytest tests/test_fm_lcb_gpu.py -q -rA -p no:cacheprovider > gpurun_out/r28_fm.log 2>&1
echo "fm rc=$?" >> gpurun_out/r28_fm.log
grep -q "fm rc=0" gpurun_out/r28_fm.log || exit 0
timeout 300 python scripts/fm_bench.py large > gpurun_out/r28_bench_pair.log 2>&1
LATTICE_FM_PAIR=0 timeout 300 python scripts/fm_bench.py large > gpurun_out/r28_bench_single.log 2>&1
LATTICE_FM_TRACE=1 timeout 120 python scripts/fm_bench.py large > gpurun_out/r28_trace.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fm_lcb_pair -c 1 -o gpurun_out/r28_pair \
  python scripts/fm_bench.py large > gpurun_out/r28_ncu.log 2>&1
echo done
